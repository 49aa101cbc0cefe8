"""ctypes binding of the C oracle (oracle/ssj_oracle.c) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker.  The product library
never calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libssjoin_ref.so")

PAIR_DTYPE = np.dtype([("id_r", "<u4"), ("id_s", "<u4"), ("overlap", "<i8")])
COUNTER_FIELDS = ("candidates", "pruned_bitmap", "bitmap_tested", "verified", "matched",
                  "saturated_records")
INT64_MAX = (1 << 63) - 1


class _Counters(C.Structure):
    _fields_ = [(f, C.c_uint64) for f in COUNTER_FIELDS]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.oracle_par_bitmap_join.argtypes = [P, P, C.c_size_t, C.c_int64, C.c_int64, C.c_int,
                                             C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                             C.c_size_t, C.c_size_t, C.POINTER(P),
                                             C.POINTER(C.c_size_t), C.POINTER(_Counters)]
        L.oracle_par_bitmap_join_store.argtypes = [P, P, C.c_size_t, C.c_int64, C.c_int64, C.c_int,
                                                   C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                                   C.c_size_t, C.c_size_t, P, C.POINTER(P),
                                                   C.POINTER(C.c_size_t), C.POINTER(_Counters)]
        L.oracle_naive_join.argtypes = [P, P, C.c_size_t, C.c_int64, C.c_int64, C.POINTER(P),
                                        C.POINTER(C.c_size_t), C.POINTER(_Counters)]
        L.oracle_naive_join_sim.argtypes = [P, P, C.c_size_t, P, P, C.c_size_t, C.c_int, C.c_int,
                                            C.c_int64, C.c_int64, C.POINTER(P),
                                            C.POINTER(C.c_size_t), C.POINTER(_Counters)]
        L.oracle_required_overlap_sim.argtypes = [C.c_int] + [C.c_int64] * 4
        L.oracle_required_overlap_sim.restype = C.c_int64
        L.oracle_build_bitmaps.argtypes = [P, P, C.c_size_t, C.c_int, C.c_int, C.c_int, P]
        L.oracle_build_row.argtypes = [P, P, C.c_size_t, C.c_int, C.c_int, C.c_int]
        L.oracle_canonicalize.argtypes = [P, P, C.c_size_t, P, P]
        L.oracle_required_overlap.argtypes = [C.c_int64] * 4
        L.oracle_required_overlap.restype = C.c_int64
        L.oracle_verify.argtypes = [P, C.c_size_t, P, C.c_size_t, C.c_int64,
                                    C.POINTER(C.c_int64)]
        L.oracle_expected_bound.argtypes = [C.c_int, C.c_int, C.c_int64]
        L.oracle_expected_bound.restype = C.c_double
        L.oracle_cutoff.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int]
        L.oracle_cutoff.restype = C.c_int64
        L.oracle_hash_token.argtypes = [C.c_uint32, C.c_int, C.c_int]
        L.oracle_hash_token.restype = C.c_uint32
        L.oracle_free.argtypes = [P]
        _lib = L
    return _lib


def _csr(tokens, offsets):
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    o = np.ascontiguousarray(offsets, dtype=np.uint64)
    if t.size == 0:
        t = np.zeros(1, dtype=np.uint32)
    return t, o


def _take_pairs(ptr, n):
    L = lib()
    if n:
        raw = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), (n * 16,))
        pairs = raw.view(PAIR_DTYPE).copy()
    else:
        pairs = np.zeros(0, dtype=PAIR_DTYPE)
    L.oracle_free(ptr)
    return pairs


def par_bitmap_join(tokens, offsets, p, q, bitmap_enabled=True, method=1, width=64, hash=0,
                    cutoff=INT64_MAX, capacity=2048, row_begin=0, row_end=0):
    t, o = _csr(tokens, offsets)
    ptr, n, cnt = C.c_void_p(), C.c_size_t(), _Counters()
    rc = lib().oracle_par_bitmap_join(t.ctypes.data, o.ctypes.data, len(o) - 1, p, q,
                                      int(bool(bitmap_enabled)), method, width, hash, cutoff,
                                      capacity, row_begin, row_end, C.byref(ptr), C.byref(n),
                                      C.byref(cnt))
    if rc != 0:
        raise RuntimeError("oracle_par_bitmap_join failed")
    return _take_pairs(ptr, n.value), {f: int(getattr(cnt, f)) for f in COUNTER_FIELDS}


def par_bitmap_join_store(tokens, offsets, store, p, q, method=1, width=64, hash=0,
                          cutoff=INT64_MAX, capacity=2048, row_begin=0, row_end=0):
    """par_bitmap_join over rows [row_begin, row_end) with a prebuilt sketch
    store (build_bitmaps of the whole collection): one build per join."""
    t, o = _csr(tokens, offsets)
    st = np.ascontiguousarray(store, dtype=np.uint64)
    ptr, n, cnt = C.c_void_p(), C.c_size_t(), _Counters()
    rc = lib().oracle_par_bitmap_join_store(t.ctypes.data, o.ctypes.data, len(o) - 1, p, q, 1, method, width,
                                            hash, cutoff, capacity, row_begin, row_end, st.ctypes.data,
                                            C.byref(ptr), C.byref(n), C.byref(cnt))
    if rc != 0:
        raise RuntimeError("oracle_par_bitmap_join_store failed")
    return _take_pairs(ptr, n.value), {f: int(getattr(cnt, f)) for f in COUNTER_FIELDS}


def naive_join(tokens, offsets, p, q):
    t, o = _csr(tokens, offsets)
    ptr, n, cnt = C.c_void_p(), C.c_size_t(), _Counters()
    if lib().oracle_naive_join(t.ctypes.data, o.ctypes.data, len(o) - 1, p, q, C.byref(ptr),
                               C.byref(n), C.byref(cnt)) != 0:
        raise RuntimeError("oracle_naive_join failed")
    return _take_pairs(ptr, n.value), {f: int(getattr(cnt, f)) for f in COUNTER_FIELDS}


def naive_join_sim(tokens, offsets, sim, p, q, s_tokens=None, s_offsets=None):
    """NAIVE self-join (s_* None) or R x S join with any similarity
    (reference src/join.cpp:91-126; sim 0 overlap, 1 jaccard, 2 cosine, 3 dice)."""
    t, o = _csr(tokens, offsets)
    self_join = s_tokens is None
    st, so = (t, o) if self_join else _csr(s_tokens, s_offsets)
    ptr, n, cnt = C.c_void_p(), C.c_size_t(), _Counters()
    if lib().oracle_naive_join_sim(t.ctypes.data, o.ctypes.data, len(o) - 1, st.ctypes.data,
                                   so.ctypes.data, len(so) - 1, 1 if self_join else 0, sim, p, q,
                                   C.byref(ptr), C.byref(n), C.byref(cnt)) != 0:
        raise RuntimeError("oracle_naive_join_sim failed")
    return _take_pairs(ptr, n.value), {f: int(getattr(cnt, f)) for f in COUNTER_FIELDS}


def required_overlap_sim(sim, p, q, sr, ss):
    return int(lib().oracle_required_overlap_sim(sim, p, q, sr, ss))


def build_bitmaps(tokens, offsets, method, width, hash=0):
    t, o = _csr(tokens, offsets)
    n = len(o) - 1
    out = np.zeros(max(n, 1) * (width // 64), dtype=np.uint64)
    lib().oracle_build_bitmaps(t.ctypes.data, o.ctypes.data, n, method, width, hash,
                               out.ctypes.data)
    return out[: n * (width // 64)]


def build_row(tokens, method, width, hash=0):
    t = np.ascontiguousarray(tokens, dtype=np.uint32)
    if t.size == 0:
        t0 = np.zeros(1, dtype=np.uint32)
    else:
        t0 = t
    row = np.zeros(width // 64, dtype=np.uint64)
    lib().oracle_build_row(row.ctypes.data, t0.ctypes.data, t.size, method, width, hash)
    return row


def canonicalize(tokens, offsets):
    t, o = _csr(tokens, offsets)
    n = len(o) - 1
    ot = np.zeros(max(int(o[-1]) if n else 0, 1), dtype=np.uint32)
    oo = np.zeros(n + 1, dtype=np.uint64)
    lib().oracle_canonicalize(t.ctypes.data, o.ctypes.data, n, ot.ctypes.data, oo.ctypes.data)
    return ot[: int(oo[-1])], oo


def required_overlap(p, q, sr, ss):
    return int(lib().oracle_required_overlap(p, q, sr, ss))


def verify(a, b, minov):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    a0 = a if a.size else np.zeros(1, dtype=np.uint32)
    b0 = b if b.size else np.zeros(1, dtype=np.uint32)
    ov = C.c_int64()
    m = lib().oracle_verify(a0.ctypes.data, a.size, b0.ctypes.data, b.size, minov, C.byref(ov))
    return bool(m), int(ov.value)


def expected_bound(method, b, n):
    return float(lib().oracle_expected_bound(method, b, n))


def cutoff(method, b, num, den, jaccard_space=True):
    return int(lib().oracle_cutoff(method, b, num, den, int(bool(jaccard_space))))


def hash_token(t, width, hash=0):
    return int(lib().oracle_hash_token(t, width, hash))


def ref_lib():
    """The UNMODIFIED reference compiled by oracle/Makefile (None when absent)."""
    if not os.path.exists(REF_LIB_PATH):
        return None
    import sys
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_1711_07295_b200 import capi
    return capi.bind(C.CDLL(REF_LIB_PATH))
