"""Python mirror of the reference's C interface for the Bitmap-Filter join.

Thin, typed wrappers over the ``ssj_*`` C ABI (reference include/ssjoin.h,
src/capi.cpp): :class:`Collection` (load / generate / write / stats),
:func:`default_options` (``ssj_join_options_init``), :func:`join`
(``ssj_join``) returning a :class:`Report` (pairs, counters, timings,
saturated_records) and the analytics helpers.  Errors surface exactly as the
C ABI reports them -- status code plus ``ssj_last_error()`` -- as
:class:`SsjError`.

The same wrappers drive any library exporting that surface; the B200 product
is :func:`paper_1711_07295_b200.load_library` (the CUDA build, which fails
loudly when it or a GPU is missing).  Tests additionally point them at the
compiled reference under ``oracle/_ref`` to compare the two.
"""
from __future__ import annotations

import ctypes as C
import os
import tempfile
from dataclasses import dataclass, field

import numpy as np

from . import capi

PAIR_DTYPE = np.dtype([("id_r", "<u4"), ("id_s", "<u4"), ("overlap", "<i8")])

STATUS_NAMES = {
    capi.SSJ_ERROR_INVALID_ARGUMENT: "INVALID_ARGUMENT",
    capi.SSJ_ERROR_IO: "IO",
    capi.SSJ_ERROR_PARSE: "PARSE",
    capi.SSJ_ERROR_INTERNAL: "INTERNAL",
}


class SsjError(RuntimeError):
    """A non-OK ``ssj_status`` with the library's thread-local message."""

    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


def _check(lib, status: int) -> None:
    if status != capi.SSJ_OK:
        raise SsjError(status, (lib.ssj_last_error() or b"").decode(errors="replace"))


def _has(lib, name: str) -> bool:
    try:
        getattr(lib, name)
        return True
    except AttributeError:
        return False


class Collection:
    """Owning wrapper of an ``ssj_collection*`` handle."""

    def __init__(self, lib, handle: int):
        self.lib = lib
        self.handle = C.c_void_p(handle)

    # ---- construction (reference include/ssjoin.h:35-59) ----
    @classmethod
    def load(cls, lib, path: str, input_format: int = capi.SSJ_INPUT_TOKEN_IDS,
             qgram_size: int = 0) -> "Collection":
        out = C.c_void_p()
        _check(lib, lib.ssj_collection_load(os.fsencode(path), input_format, qgram_size,
                                            C.byref(out)))
        return cls(lib, out.value)

    @classmethod
    def generate(cls, lib, num_sets: int, mean_size: float, universe: int, seed: int = 0,
                 distribution: int = capi.SSJ_DIST_UNIFORM,
                 zipf_exponent: float = 0.0) -> "Collection":
        cfg = capi.GeneratorConfig(distribution, num_sets, mean_size, universe, seed,
                                   zipf_exponent)
        out = C.c_void_p()
        _check(lib, lib.ssj_collection_generate(C.byref(cfg), C.byref(out)))
        return cls(lib, out.value)

    @classmethod
    def from_records(cls, lib, records) -> "Collection":
        """Canonical collection from raw token-id records (ids taken as-is)."""
        lens = np.fromiter((len(r) for r in records), dtype=np.uint64, count=len(records))
        offsets = np.zeros(len(records) + 1, dtype=np.uint64)
        np.cumsum(lens, out=offsets[1:])
        tokens = (np.concatenate([np.asarray(r, dtype=np.uint32) for r in records])
                  if len(records) and offsets[-1] else np.zeros(0, dtype=np.uint32))
        return cls.from_csr(lib, tokens, offsets)

    @classmethod
    def from_csr(cls, lib, tokens: np.ndarray, offsets: np.ndarray) -> "Collection":
        tokens = np.ascontiguousarray(tokens, dtype=np.uint32)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = len(offsets) - 1
        if _has(lib, "ssjb_collection_from_csr"):
            out = C.c_void_p()
            _check(lib, lib.ssjb_collection_from_csr(tokens.ctypes.data, offsets.ctypes.data, n,
                                                      C.byref(out)))
            return cls(lib, out.value)
        # A library with only the reference surface: go through an id file.
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "coll.txt")
            write_id_file(path, tokens, offsets)
            return cls.load(lib, path)

    def write(self, path: str) -> None:
        _check(self.lib, self.lib.ssj_collection_write(self.handle, os.fsencode(path)))

    def csr(self):
        """(tokens u32, offsets u64) of the canonical collection."""
        lib = self.lib
        if _has(lib, "ssjb_collection_csr"):
            tp, op, n = C.c_void_p(), C.c_void_p(), C.c_size_t()
            _check(lib, lib.ssjb_collection_csr(self.handle, C.byref(tp), C.byref(op), C.byref(n)))
            nn = n.value
            offsets = np.ctypeslib.as_array(C.cast(op, C.POINTER(C.c_uint64)), (nn + 1,)).copy()
            total = int(offsets[-1])
            tokens = (np.ctypeslib.as_array(C.cast(tp, C.POINTER(C.c_uint32)), (total,)).copy()
                      if total else np.zeros(0, dtype=np.uint32))
            return tokens, offsets
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "coll.txt")
            self.write(path)
            return read_id_file(path)

    # ---- stats (reference include/ssjoin.h:41-45) ----
    def __len__(self):
        return int(self.lib.ssj_collection_size(self.handle))

    @property
    def median_size(self):
        return int(self.lib.ssj_collection_median_size(self.handle))

    @property
    def mean_size(self):
        return float(self.lib.ssj_collection_mean_size(self.handle))

    @property
    def max_size(self):
        return int(self.lib.ssj_collection_max_size(self.handle))

    @property
    def universe(self):
        return int(self.lib.ssj_collection_universe(self.handle))

    def close(self):
        if self.handle is not None and self.handle.value:
            self.lib.ssj_collection_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_options(lib, **overrides) -> capi.JoinOptions:
    """``ssj_join_options_init`` defaults (reference src/capi.cpp:201-215) + overrides."""
    opts = capi.JoinOptions()
    lib.ssj_join_options_init(C.byref(opts))
    for k, v in overrides.items():
        if k == "threshold":
            num, den = v
            opts.threshold_num, opts.threshold_den = num, den
        else:
            setattr(opts, k, v)
    return opts


def par_bitmap_options(lib, threshold=(9, 10), method=capi.SSJ_BITMAP_XOR, bits=64,
                       cutoff_mode=capi.SSJ_CUTOFF_OFF, **kw) -> capi.JoinOptions:
    """Options for SSJ_ALGO_PAR_BITMAP as the reference CLI sets them
    (tools/ssjoin_cli.cpp:153-165: Xor, cutoff OFF)."""
    return default_options(lib, algorithm=capi.SSJ_ALGO_PAR_BITMAP, threshold=threshold,
                           bitmap_enabled=1, bitmap_method=method, bitmap_bits=bits,
                           cutoff_mode=cutoff_mode, **kw)


@dataclass
class Report:
    pairs: np.ndarray
    counters: dict
    timings: dict
    saturated_records: int
    extra: dict = field(default_factory=dict)


class _ReportOwner:
    """Frees an ``ssj_report`` when the last numpy view of its pairs is gone."""

    def __init__(self, lib, handle):
        self.lib, self.handle = lib, handle

    def __del__(self):
        try:
            self.lib.ssj_report_free(self.handle)
        except Exception:
            pass


_ZERO_COPY_PAIRS = 1 << 20  # larger results are viewed in place, not copied


def _take_report(lib, handle) -> Report:
    n = int(lib.ssj_report_pair_count(handle))
    owner = None
    if n:
        ptr = lib.ssj_report_pairs(handle)
        if n >= _ZERO_COPY_PAIRS:
            # the report's own pair array (ssj_report_pairs, valid until
            # ssj_report_free) becomes the numpy buffer; freed with the array
            buf = (C.c_uint8 * (n * 16)).from_address(C.cast(ptr, C.c_void_p).value)
            owner = buf._owner = _ReportOwner(lib, handle)
            pairs = np.frombuffer(buf, dtype=PAIR_DTYPE)
        else:
            raw = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), (n * 16,))
            pairs = raw.view(PAIR_DTYPE).copy()
    else:
        pairs = np.zeros(0, dtype=PAIR_DTYPE)
    cnt = capi.Counters()
    lib.ssj_report_counters(handle, C.byref(cnt))
    tim = capi.Timings()
    lib.ssj_report_timings(handle, C.byref(tim))
    rep = Report(pairs=pairs,
                 counters={k: int(getattr(cnt, k)) for k, _ in capi.Counters._fields_},
                 timings={k: float(getattr(tim, k)) for k, _ in capi.Timings._fields_},
                 saturated_records=int(lib.ssj_report_saturated_records(handle)))
    if _has(lib, "ssjb_report_stats"):
        st = capi.Stats()
        if lib.ssjb_report_stats(handle, C.byref(st)) == capi.SSJ_OK:
            rep.extra = {k: (float(getattr(st, k)) if isinstance(getattr(st, k), float)
                             else int(getattr(st, k))) for k, _ in capi.Stats._fields_}
    if owner is None:
        lib.ssj_report_free(handle)
    return rep


def join(coll: Collection, opts: capi.JoinOptions, other: Collection | None = None) -> Report:
    lib = coll.lib
    out = C.c_void_p()
    _check(lib, lib.ssj_join(coll.handle, other.handle if other is not None else None,
                             C.byref(opts), C.byref(out)))
    return _take_report(lib, out)


def join_stream(coll: Collection, opts: capi.JoinOptions, on_chunk, other: Collection | None = None,
                chunk_pairs: int = 0) -> Report:
    """Streaming delivery (B200 extension, ssjb_join_stream): ``on_chunk(pairs)``
    receives consecutive chunks of the canonical pair list as numpy views
    valid only during the call (copy to keep); returning True stops the join.
    The returned report holds counters only (no pairs)."""
    lib = coll.lib
    err = []

    def sink(ptr, n, _user):
        try:
            raw = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), (n * 16,))
            return 1 if on_chunk(raw.view(PAIR_DTYPE)) else 0
        except BaseException as e:  # noqa: BLE001 -- re-raised after the C call returns
            err.append(e)
            return 1

    cb = capi.PAIR_SINK(sink)
    out = C.c_void_p()
    status = lib.ssjb_join_stream(coll.handle, other.handle if other is not None else None,
                                  C.byref(opts), chunk_pairs, cb, None, C.byref(out))
    if err:
        raise err[0]
    _check(lib, status)
    return _take_report(lib, out)


def join_count(coll: Collection, opts: capi.JoinOptions, other: Collection | None = None) -> Report:
    """Count-first (ssjb_join_count): counters incl. matched, no pairs."""
    lib = coll.lib
    out = C.c_void_p()
    _check(lib, lib.ssjb_join_count(coll.handle, other.handle if other is not None else None,
                                    C.byref(opts), C.byref(out)))
    return _take_report(lib, out)


def join_write_pairs(coll: Collection, opts: capi.JoinOptions, path: str,
                     other: Collection | None = None) -> Report:
    """Streams the pairs into ``path`` as "id_r id_s overlap" lines (ssjb_join_write_pairs)."""
    lib = coll.lib
    out = C.c_void_p()
    _check(lib, lib.ssjb_join_write_pairs(coll.handle, other.handle if other is not None else None,
                                          C.byref(opts), os.fsencode(path), C.byref(out)))
    return _take_report(lib, out)


def join_rows(coll: Collection, opts: capi.JoinOptions, row_begin: int, row_end: int,
              device: int = -1) -> Report:
    """Rows [row_begin, row_end) of a self-join (B200 extension, ssjb_join_rows)."""
    lib = coll.lib
    out = C.c_void_p()
    _check(lib, lib.ssjb_join_rows(coll.handle, C.byref(opts), row_begin, row_end, device,
                                   C.byref(out)))
    return _take_report(lib, out)


def partition_rows(coll: Collection, opts: capi.JoinOptions, parts: int) -> np.ndarray:
    bounds = np.zeros(parts + 1, dtype=np.uint64)
    _check(coll.lib, coll.lib.ssjb_partition_rows(coll.handle, C.byref(opts), parts,
                                                  bounds.ctypes.data))
    return bounds


def build_bitmaps(coll: Collection, method: int, bits: int, hash: int = 0,
                  device: int = -1) -> np.ndarray:
    """The device sketch store (B200 extension, ssjb_build_bitmaps)."""
    out = np.zeros(max(len(coll), 1) * (bits // 64), dtype=np.uint64)
    _check(coll.lib, coll.lib.ssjb_build_bitmaps(coll.handle, method, bits, hash, device,
                                                 out.ctypes.data))
    return out[: len(coll) * (bits // 64)]


def pin_device(coll: Collection, device: int = 0) -> None:
    _check(coll.lib, coll.lib.ssjb_collection_pin_device(coll.handle, device))


def unpin_device(coll: Collection, device: int = 0) -> None:
    _check(coll.lib, coll.lib.ssjb_collection_unpin_device(coll.handle, device))


def resolve_bitmap(coll: Collection, opts: capi.JoinOptions):
    lib = coll.lib
    m, b, c = C.c_int(-1), C.c_int(0), C.c_int64(0)
    _check(lib, lib.ssj_resolve_bitmap(coll.handle, C.byref(opts), C.byref(m), C.byref(b),
                                       C.byref(c)))
    return m.value, b.value, c.value


def cutoff(lib, method, bits, num, den, space=capi.SSJ_SPACE_JACCARD) -> int:
    out = C.c_int64()
    _check(lib, lib.ssj_cutoff(method, bits, num, den, space, C.byref(out)))
    return out.value


def expected_bound(lib, method, bits, n) -> float:
    out = C.c_double()
    _check(lib, lib.ssj_expected_bound(method, bits, n, C.byref(out)))
    return out.value


def parse_threshold(lib, text: str):
    num, den = C.c_int64(), C.c_int64()
    _check(lib, lib.ssj_parse_threshold(text.encode(), C.byref(num), C.byref(den)))
    return num.value, den.value


# ---- canonical id files (reference src/collection.cpp:97-137,153-168) ----

def write_id_file(path: str, tokens: np.ndarray, offsets: np.ndarray) -> None:
    with open(path, "w") as f:
        for r in range(len(offsets) - 1):
            seg = tokens[int(offsets[r]):int(offsets[r + 1])]
            f.write(" ".join(map(str, seg.tolist())))
            f.write("\n")


def read_id_file(path: str):
    toks, offs = [], [0]
    with open(path) as f:
        for line in f:
            vals = [int(x) for x in line.split()]
            toks.extend(vals)
            offs.append(len(toks))
    return np.asarray(toks, dtype=np.uint32), np.asarray(offs, dtype=np.uint64)
