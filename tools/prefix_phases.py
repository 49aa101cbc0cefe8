#!/usr/bin/env python3
"""GPU prefix-filter joins (ALLPAIRS..ADAPTJOIN, bitmap off / filter3 / filter2)
on the BASELINE-shaped collections: ssj_join seconds (second of two runs),
counters and engine phases, one JSON line per join.

    python tools/prefix_phases.py c1 c2 c3 [--algo 1 --bitmap f3 --reps 1]
"""
import json
import sys
import time

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1711_07295_b200 import capi, datasets as D, load_library  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

TAU = {"c1": (9, 10), "c2": (4, 5), "c3": (1, 2), "c4": (7, 10)}


def main(names, only_algo=None, only_bitmap=None, reps=2):
    lib = load_library()
    for name in names:
        coll = getattr(D, name)(lib)
        for algo in (1, 2, 3, 4, 5):
            for bl, kw in (("off", dict(bitmap_enabled=0)), ("f3", dict(bitmap_enabled=1)),
                           ("f2", dict(bitmap_enabled=1, placement=capi.SSJ_PLACEMENT_FILTER2))):
                if algo in (4, 5) and bl == "f2":
                    continue
                if (only_algo and algo != only_algo) or (only_bitmap and bl != only_bitmap):
                    continue
                opts = S.default_options(lib, algorithm=algo, threshold=TAU[name], **kw)
                best = None
                for _ in range(reps):
                    t = time.perf_counter()
                    rep = S.join(coll, opts)
                    dt = time.perf_counter() - t
                    best = dt if best is None else min(best, dt)
                print(json.dumps(dict(config=name, algo=algo, bitmap=bl, join_s=round(best, 4),
                                      pairs=int(len(rep.pairs)), counters=rep.counters,
                                      stats={k: rep.extra.get(k) for k in ("window_pairs", "launches", "ms_upload",
                                                                           "ms_filter", "ms_verify", "ms_sort")})),
                      flush=True)


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3"])
    ap.add_argument("--algo", type=int, default=None)
    ap.add_argument("--bitmap", default=None)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    main(a.configs, a.algo, a.bitmap, a.reps)
