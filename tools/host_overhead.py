#!/usr/bin/env python3
"""Per-join wall time vs device phases for the C2 sweep: pinned replica and
per-join upload (streamed ingest on/off).  Diagnostics for the e2e path."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

lib = pkg.load_library()
coll = D.c2(lib)
mode = sys.argv[1] if len(sys.argv) > 1 else "pinned"
if mode == "pinned":
    S.pin_device(coll, 0)
for rep in range(3):
    rows = []
    t_all = time.perf_counter()
    for tau in D.C2_TAUS:
        t0 = time.perf_counter()
        r = S.join(coll, D.c2_options(lib, tau))
        wall = (time.perf_counter() - t0) * 1e3
        dev = sum(r.extra[k] for k in r.extra if k.startswith("ms_"))
        rows.append({"tau": f"{tau[0]}/{tau[1]}", "wall": round(wall, 3), "dev": round(dev, 3),
                     "total_s": round(r.timings["total_s"] * 1e3, 3),
                     "ms": {k[3:]: round(r.extra[k], 3) for k in r.extra if k.startswith("ms_")}})
    step = (time.perf_counter() - t_all) * 1e3
print(json.dumps({"mode": mode, "env": {k: v for k, v in os.environ.items() if k.startswith("SSJB")},
                  "step_ms": round(step, 3), "joins": rows}))
