#!/usr/bin/env python3
"""Regenerates the golden fixtures under tests/golden/ from the UNMODIFIED
reference engine.

Runs only in the build container (it needs /root/reference for the bitmap
shim's headers and oracle/_ref/libssjoin_ref.so, which `make -C oracle`
compiles from the reference sources).  The GPU box never runs this; it only
reads the committed fixtures.

    python tests/golden/make_golden.py          # writes golden.json + golden_pairs.npz

What is pinned (every value comes from the reference library itself):
  * generator:   canonical-file sha256 + stats of ssj_collection_generate outputs
                 (reference src/collection.cpp:193-254), incl. config C1
  * bitmaps:     sha256 of ssj::build_bitmaps stores, Set/Xor/Next x widths x hashes
                 (reference src/bitmap.cpp:40-158)
  * joins:       pairs (or their sha256 when large), counters and saturated_records
                 of ssj_join(PAR_BITMAP) / ssj_join(NAIVE) over the reference tests'
                 own collections (test_parallel.cpp, test_joins.cpp, test_capi.cpp,
                 acceptance.cpp criteria 1 and 8) and SURVEY.md section 7.4 edge cases
  * analytics:   ssj_cutoff / ssj_expected_bound / ssj_resolve_bitmap / ssj_parse_threshold
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1711_07295_b200 import capi  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

REF_PROJ = os.environ.get("SSJ_REFERENCE", "/root/reference/proj")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libssjoin_ref.so")
OUT_DIR = os.path.dirname(os.path.abspath(__file__))
PAIR_INLINE_LIMIT = 20000


def sha(arr) -> str:
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def build_shim() -> C.CDLL:
    out = os.path.join(tempfile.gettempdir(), "ssj_ref_bitmap_shim.so")
    subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared",
                    f"-I{REF_PROJ}/src", os.path.join(OUT_DIR, "ref_bitmap_shim.cpp"),
                    REF_SO, f"-Wl,-rpath,{os.path.dirname(REF_SO)}", "-o", out], check=True)
    lib = C.CDLL(out)
    lib.ref_build_bitmaps.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int,
                                      C.c_int, C.c_void_p]
    return lib


def main() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True)
    ref = capi.bind(C.CDLL(REF_SO))
    shim = build_shim()
    golden = {"generator": [], "bitmaps": [], "joins": [], "analytics": {}}
    pairs_store = {}
    collections = {}

    def gen(name, num_sets, mean, universe, seed, dist=capi.SSJ_DIST_UNIFORM, zexp=0.0,
            keep=True):
        coll = S.Collection.generate(ref, num_sets, mean, universe, seed, dist, zexp)
        t, o = coll.csr()
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "c.txt")
            coll.write(p)
            digest = hashlib.sha256(open(p, "rb").read()).hexdigest()
        golden["generator"].append(dict(
            name=name, distribution=dist, num_sets=num_sets, mean_size=mean, universe=universe,
            seed=seed, zipf_exponent=zexp, file_sha256=digest, size=len(coll),
            median=coll.median_size, mean=coll.mean_size, max=coll.max_size,
            universe_size=coll.universe))
        if keep:
            collections[name] = (t, o)
            pairs_store[f"coll/{name}/tokens"] = t
            pairs_store[f"coll/{name}/offsets"] = o
        return coll

    def explicit(name, records):
        coll = S.Collection.from_records(ref, records)
        t, o = coll.csr()
        collections[name] = (t, o)
        pairs_store[f"coll/{name}/tokens"] = t
        pairs_store[f"coll/{name}/offsets"] = o
        return coll

    # ---- collections (reference tests' own fixtures) ----
    cols = {}
    cols["par_1500"] = gen("par_1500", 1500, 8, 150, 8)        # test_parallel.cpp:22
    cols["par_1200"] = gen("par_1200", 1200, 9, 100, 9)        # test_parallel.cpp:38
    cols["par_800"] = gen("par_800", 800, 8, 60, 10)           # test_parallel.cpp:62
    cols["par_500"] = gen("par_500", 500, 8, 60, 12)           # test_parallel.cpp:102
    cols["capi_400"] = gen("capi_400", 400, 8, 80, 4)          # test_capi.cpp:42-48
    cols["hash_300"] = gen("hash_300", 300, 8, 70, 123)        # test_joins.cpp:132
    cols["det_400"] = gen("det_400", 400, 7, 70, 91)           # test_joins.cpp:194
    cols["acc8_2000"] = gen("acc8_2000", 2000, 10, 60, 777)    # acceptance.cpp:299
    cols["wide_300"] = gen("wide_300", 300, 100, 4000, 9)      # test_capi.cpp:113-119
    cols["zipf_3000"] = gen("zipf_3000", 3000, 20, 2000, 5, capi.SSJ_DIST_ZIPF)
    cols["zipf_big_1500"] = gen("zipf_big_1500", 1500, 70, 800, 6, capi.SSJ_DIST_ZIPF)
    for c in range(20):                                        # acceptance.cpp:69-73
        universe = (50, 500, 5000)[c % 3]
        sets = 1200 if universe == 50 else 2000
        cols[f"acc1_{c}"] = gen(f"acc1_{c}", sets, 10, universe, 100 + c)
    gen("C1", 100000, 10, 220, 1, keep=False)                  # BASELINE config 1
    gen("gen_zipf_alt_exp", 5000, 12, 41275, 3, capi.SSJ_DIST_ZIPF, 1.3, keep=False)
    gen("gen_small_universe", 2000, 30, 25, 11, keep=False)    # sizes clipped to universe

    cols["dups_2500"] = explicit("dups_2500", [[1, 2, 3, 4, 5]] * 2500)  # test_parallel.cpp:76
    cols["edge_empty"] = explicit("edge_empty", [[]] * 5 + [[1, 2, 3], [1, 2, 3], [4, 5],
                                                           [4, 5, 6], [1, 2, 3, 4]])
    cols["three"] = explicit("three", [[1, 2, 3], [1, 2, 3, 4], [5, 6, 7]])  # test_joins.cpp:25
    cols["clones5"] = explicit("clones5", [[7, 8, 9]] * 5)                  # test_joins.cpp:43
    cols["single"] = explicit("single", [[5, 6]])
    cols["empty"] = explicit("empty", [])
    cols["pair2"] = explicit("pair2", [[1, 2], [1, 2, 3]])

    # ---- bitmaps ----
    for name in ("par_1500", "zipf_3000", "zipf_big_1500", "wide_300", "edge_empty", "acc1_1"):
        t, o = collections[name]
        n = len(o) - 1
        for width in (64, 128, 192, 256, 512):
            for method in (0, 1, 2):
                for h in (0, 1):
                    out = np.zeros(max(n, 1) * (width // 64), dtype=np.uint64)
                    tt = t if t.size else np.zeros(1, dtype=np.uint32)
                    shim.ref_build_bitmaps(tt.ctypes.data, o.ctypes.data, n, method, width, h,
                                           out.ctypes.data)
                    golden["bitmaps"].append(dict(collection=name, method=method, width=width,
                                                  hash=h, sha256=sha(out[: n * (width // 64)])))

    # ---- joins ----
    case_id = [0]

    def run(coll_name, label, **kw):
        coll = cols[coll_name]
        opts = S.default_options(ref, **kw)
        rep = S.join(coll, opts)
        cid = f"j{case_id[0]:04d}"
        case_id[0] += 1
        entry = dict(id=cid, collection=coll_name, label=label,
                     options={k: getattr(opts, k) for k, _ in capi.JoinOptions._fields_},
                     counters=rep.counters, saturated_records=rep.saturated_records,
                     pair_count=int(len(rep.pairs)), pairs_sha256=sha(rep.pairs))
        if len(rep.pairs) <= PAIR_INLINE_LIMIT:
            pairs_store[f"pairs/{cid}"] = rep.pairs
        golden["joins"].append(entry)
        return rep

    PB = capi.SSJ_ALGO_PAR_BITMAP
    X, OFF = capi.SSJ_BITMAP_XOR, capi.SSJ_CUTOFF_OFF
    for tau in ((1, 2), (7, 10), (9, 10)):                      # test_parallel.cpp:21-35
        for workers in (1, 8):
            run("par_1500", "test_parallel oracle equality", algorithm=PB, threshold=tau,
                bitmap_enabled=1, bitmap_method=X, cutoff_mode=OFF, workers=workers)
        run("par_1500", "naive oracle", algorithm=capi.SSJ_ALGO_NAIVE, threshold=tau)
    run("par_1200", "worker invariance", algorithm=PB, threshold=(3, 5), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF, workers=4)
    run("par_800", "capacity 1", algorithm=PB, threshold=(1, 2), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF, workers=4, buffer_capacity=1)
    run("par_800", "capacity 3", algorithm=PB, threshold=(1, 2), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF, buffer_capacity=3)
    run("par_800", "capacity 17 next", algorithm=PB, threshold=(1, 2), bitmap_enabled=1,
        bitmap_method=capi.SSJ_BITMAP_NEXT, cutoff_mode=OFF, buffer_capacity=17)
    run("dups_2500", "2500 identical records overflow the buffer", algorithm=PB,
        threshold=(9, 10), bitmap_enabled=1, bitmap_method=X, cutoff_mode=OFF, workers=4)
    run("par_500", "bitmap disabled", algorithm=PB, threshold=(7, 10), bitmap_enabled=0)
    run("par_500", "bitmap disabled cap 5", algorithm=PB, threshold=(7, 10), bitmap_enabled=0,
        buffer_capacity=5)
    run("capi_400", "test_capi par-bitmap", algorithm=PB, threshold=(7, 10), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF, workers=4)
    run("capi_400", "test_capi naive", algorithm=capi.SSJ_ALGO_NAIVE, threshold=(7, 10))
    run("hash_300", "multiplicative hash", algorithm=PB, threshold=(3, 5), bitmap_enabled=1,
        bitmap_hash=capi.SSJ_HASH_MULT, cutoff_mode=OFF)
    for tau in ((7, 10), (1, 2), (4, 5)):
        run("det_400", "default combined + auto cutoff", algorithm=PB, threshold=tau,
            bitmap_enabled=1)
    for cap in (2048, 1):                                       # acceptance.cpp:297-336
        run("acc8_2000", "acceptance criterion 8", algorithm=PB, threshold=(3, 5),
            bitmap_enabled=1, bitmap_method=X, cutoff_mode=OFF, workers=4,
            buffer_capacity=cap)
    run("wide_300", "auto width 128 combined auto cutoff", algorithm=PB, threshold=(9, 10),
        bitmap_enabled=1)
    for width in (64, 128, 192, 256, 512):
        for method in (0, 1, 2):
            for h in (0, 1):
                run("zipf_big_1500", "width/method/hash grid", algorithm=PB, threshold=(1, 2),
                    bitmap_enabled=1, bitmap_method=method, bitmap_bits=width, bitmap_hash=h,
                    cutoff_mode=OFF, buffer_capacity=64)
    for width in (64, 256):
        run("zipf_3000", "auto cutoff", algorithm=PB, threshold=(7, 10), bitmap_enabled=1,
            bitmap_method=X, bitmap_bits=width, cutoff_mode=capi.SSJ_CUTOFF_AUTO)
        run("zipf_3000", "explicit cutoff", algorithm=PB, threshold=(3, 5), bitmap_enabled=1,
            bitmap_method=capi.SSJ_BITMAP_SET, bitmap_bits=width,
            cutoff_mode=capi.SSJ_CUTOFF_EXPLICIT, cutoff_value=20)
    for tau in ((1, 1), (1, 2)):                                # SURVEY 7.4 edge cases
        for en in (1, 0):
            run("edge_empty", "empty records / tau=1", algorithm=PB, threshold=tau,
                bitmap_enabled=en, bitmap_method=X, cutoff_mode=OFF, buffer_capacity=2)
    run("three", "three-record", algorithm=PB, threshold=(7, 10), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF)
    run("three", "three-record naive", algorithm=capi.SSJ_ALGO_NAIVE, threshold=(7, 10))
    run("clones5", "clones tau=1", algorithm=PB, threshold=(1, 1), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF)
    run("clones5", "clones tau=1 naive", algorithm=capi.SSJ_ALGO_NAIVE, threshold=(1, 1))
    run("single", "single record", algorithm=PB, threshold=(1, 2), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF)
    run("empty", "empty collection", algorithm=PB, threshold=(1, 2), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF)
    run("pair2", "two records", algorithm=PB, threshold=(1, 2), bitmap_enabled=1,
        bitmap_method=X, cutoff_mode=OFF)
    taus = ((1, 2), (3, 5), (7, 10), (3, 4), (4, 5), (17, 20), (9, 10), (19, 20))
    for c in range(20):                                         # acceptance.cpp:65-120
        for tau in taus:
            for bm in range(5):
                kw = dict(algorithm=PB, threshold=tau, cutoff_mode=OFF)
                if bm > 0:
                    kw.update(bitmap_enabled=1, bitmap_method=bm - 1)
                run(f"acc1_{c}", "acceptance criterion 1", **kw)

    # ---- analytics / host resolution ----
    an = golden["analytics"]
    an["cutoff"] = []
    for method in (0, 1, 2):
        for bits in (64, 128, 192, 256, 512, 1024):
            for tau in ((1, 2), (3, 5), (7, 10), (4, 5), (9, 10), (19, 20), (1, 1), (72, 100)):
                for space in (0, 1):
                    an["cutoff"].append(dict(method=method, bits=bits, num=tau[0], den=tau[1],
                                             space=space,
                                             value=S.cutoff(ref, method, bits, *tau, space)))
    an["expected_bound"] = [dict(method=m, bits=b, n=n, value=S.expected_bound(ref, m, b, n))
                            for m in (0, 1, 2) for b in (64, 128, 256) for n in (0, 1, 8, 33, 500)]
    an["resolve"] = []
    for name in ("par_1500", "wide_300", "zipf_big_1500", "edge_empty"):
        for tau in ((1, 2), (3, 5), (9, 10)):
            for method in (0, 1, 2, 3):
                for mode in (0, 1, 2):
                    opts = S.default_options(ref, algorithm=PB, threshold=tau, bitmap_enabled=1,
                                             bitmap_method=method, cutoff_mode=mode,
                                             cutoff_value=42)
                    an["resolve"].append(dict(collection=name, num=tau[0], den=tau[1],
                                              method=method, cutoff_mode=mode,
                                              result=list(S.resolve_bitmap(cols[name], opts))))
    an["parse"] = []
    for text in ("0.6", "3/4", "7", "x", "0.75", "1", "1/1", "2/4", ".5", "5.", "0.123456789",
                 "0.1234567891", "3/0", "", "1/2/3", "-1", "1234567890123456789", "9/10"):
        try:
            an["parse"].append(dict(text=text, ok=True, value=list(S.parse_threshold(ref, text))))
        except S.SsjError as e:
            an["parse"].append(dict(text=text, ok=False, status=e.status))

    with open(os.path.join(OUT_DIR, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1)
    np.savez_compressed(os.path.join(OUT_DIR, "golden_pairs.npz"), **pairs_store)
    print(f"wrote {len(golden['joins'])} joins, {len(golden['bitmaps'])} bitmap stores, "
          f"{len(golden['generator'])} generator fingerprints")


if __name__ == "__main__":
    main()
