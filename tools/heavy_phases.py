#!/usr/bin/env python3
"""Phase breakdown of one full-size join per heavy BASELINE config (C3/C4/C5)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

lib = pkg.load_library()
names = sys.argv[1:] or ["C3", "C5", "C4"]
for name in names:
    mk, mo, kw = {"C3": (D.c3, D.c3_options, {}), "C4": (D.c4, D.c4_options, {}),
                  "C4_b128": (D.c4, D.c4_options, {"bits": 128}), "C5": (D.c5, D.c5_options, {})}[name]
    t0 = time.perf_counter()
    coll = mk(lib)
    gen = time.perf_counter() - t0
    for rep in range(2):
        t0 = time.perf_counter()
        r = S.join(coll, mo(lib, **kw))
        wall = time.perf_counter() - t0
    x = r.extra
    print(json.dumps({"config": name, "gen_s": round(gen, 2), "wall_s": round(wall, 3),
                      "window": r.counters["candidates"], "verified": r.counters["verified"],
                      "matched": r.counters["matched"], "saturated": r.saturated_records,
                      "survivors_emitted": x["survivors"], "head_survivors": x.get("head_survivors"),
                      "head_k": x.get("head_k"), "batches": x["batches"], "kernel": x["filter_kernel"],
                      "ms": {k[3:]: round(x[k], 2) for k in x if k.startswith("ms_")},
                      "timings": r.timings}), flush=True)
    del coll
