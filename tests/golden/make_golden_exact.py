#!/usr/bin/env python3
"""Full-size ground truth for the configs PAR_BITMAP cannot finish on the CPU
(C4 ORKUT-shaped, C5 AOL-shaped): the UNMODIFIED reference's exact
prefix-filter join (oracle/_ref/libssjoin_ref.so, ``ssj_join`` with
SSJ_ALGO_PPJOIN by default) run in the build container.

Every exact algorithm of the reference returns the same pair list as
PAR_BITMAP -- same (id_r, id_s) set, same overlaps, canonical order
(reference proj/tests/test_joins.cpp:62-112 asserts exactly this) -- while
its counters are algorithm-specific.  So these fixtures pin the pairs
(``pair_count``, ``pairs_sha256`` over the 16-byte ``ssj_pair`` records in
canonical order) and the collection (``collection_sha256``); PAR_BITMAP's
counters stay pinned by the row-block samples in tests/test_gpu_heavy.py.

Appends one JSON line per case to tests/golden/large.jsonl (case name
``<config>_exact``; the same pairs hold for every bitmap width, so C4 and
C4_b128 share ``C4_exact``); existing cases are skipped.

    python tests/golden/make_golden_exact.py [C4] [C5] [--algo ppjoin|allpairs|groupjoin]
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1711_07295_b200 import capi, datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "large.jsonl")
ALGOS = {"ppjoin": capi.SSJ_ALGO_PPJOIN, "allpairs": capi.SSJ_ALGO_ALLPAIRS,
         "groupjoin": capi.SSJ_ALGO_GROUPJOIN}
CASES = {"C4": (D.c4, (7, 10)), "C5": (D.c5, (4, 5)), "C3": (D.c3, (1, 2))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["C4", "C5"])
    ap.add_argument("--algo", default="ppjoin", choices=sorted(ALGOS))
    a = ap.parse_args()
    ref = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libssjoin_ref.so")))
    done = set()
    if os.path.exists(OUT):
        for line in open(OUT):
            done.add(json.loads(line)["case"])
    for name in a.cases:
        case = f"{name}_exact"
        if case in done:
            print(case, "already present", flush=True)
            continue
        mk, tau = CASES[name]
        coll = mk(ref)
        t, o = coll.csr()
        # Jaccard, bitmap filter off: the reference's plain exact algorithm
        opts = S.default_options(ref, algorithm=ALGOS[a.algo], threshold=tau, bitmap_enabled=0)
        t0 = time.time()
        rep = S.join(coll, opts)
        wall = time.time() - t0
        pairs = rep.pairs
        key = pairs["id_r"].astype(np.uint64) << np.uint64(32) | pairs["id_s"].astype(np.uint64)
        if len(key) > 1 and not (key[1:] > key[:-1]).all():
            pairs = pairs[np.argsort(key, kind="stable")]
        entry = dict(case=case, tau=list(tau), algorithm=a.algo,
                     collection_sha256=hashlib.sha256(t.tobytes() + o.tobytes()).hexdigest(),
                     pair_count=int(len(pairs)),
                     pairs_sha256=hashlib.sha256(pairs.tobytes()).hexdigest(),
                     overlap_sum=int(pairs["overlap"].astype(np.int64).sum()),
                     ref_counters=rep.counters, ref_total_s=rep.timings["total_s"], ref_wall_s=wall,
                     note="pairs only: counters are algorithm-specific (test_joins.cpp:62-112)")
        with open(OUT, "a") as f:
            f.write(json.dumps(entry) + "\n")
        print(case, len(pairs), f"{wall:.1f}s", flush=True)
        del pairs, rep, coll


if __name__ == "__main__":
    main()
