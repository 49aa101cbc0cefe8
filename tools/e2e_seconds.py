#!/usr/bin/env python3
"""End-to-end ssj_join seconds (host collection in, sorted pairs out; the
reference's total_s boundary) for the BASELINE configs, best of 3."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import load_library, ssjoin as S  # noqa: E402

lib = load_library()
cases = [("C1", D.c1, lambda: [D.c1_options(lib)]),
         ("C2", D.c2, lambda: [D.c2_options(lib, t) for t in ((1, 2), (7, 10), (9, 10))]),
         ("C3", D.c3, lambda: [D.c3_options(lib)]),
         ("C4", D.c4, lambda: [D.c4_options(lib)]),
         ("C5", D.c5, lambda: [D.c5_options(lib)])]
only = set(sys.argv[1:])
for name, mk, opts in cases:
    if only and name not in only:
        continue
    coll = mk(lib)
    for o in opts():
        best, rep = None, None
        for _ in range(3):
            t0 = time.perf_counter()
            rep = S.join(coll, o)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        print(json.dumps({"config": name, "tau": f"{o.threshold_num}/{o.threshold_den}", "bits": o.bitmap_bits,
                          "e2e_s": round(best, 4), "window_pairs": rep.counters["candidates"],
                          "matched": rep.counters["matched"],
                          "G_pair_cmp_per_s": round(rep.counters["candidates"] / best / 1e9, 1)}), flush=True)
    del coll
