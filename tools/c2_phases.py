#!/usr/bin/env python3
"""Per-threshold phase breakdown of the C2 sweep (diagnostics for profiles/)."""
import json
import time
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lib = pkg.load_library()
coll = D.c2(lib)
S.pin_device(coll, 0)
for tau in D.C2_TAUS:
    for _ in range(reps):
        t0 = time.perf_counter()
        r = S.join(coll, D.c2_options(lib, tau, bits=bits))
        wall = (time.perf_counter() - t0) * 1e3
    x = r.extra
    print(json.dumps({"tau": f"{tau[0]}/{tau[1]}", "bits": bits, "window": r.counters["candidates"],
                      "survivors": x["survivors"], "matched": r.counters["matched"],
                      "saturated": r.saturated_records, "batches": x["batches"],
                      "ms": {k[3:]: round(x[k], 3) for k in x if k.startswith("ms_")},
                      "wall_ms": round(wall, 3), "total_s_ms": round(r.timings["total_s"] * 1e3, 3),
                      "launches": x["launches"], "kernel": x["filter_kernel"],
                      "filter_Gpair_s": round(r.counters["candidates"] / x["ms_filter"] / 1e6, 1),
                      "verify_Mpair_s": round(x["survivors"] / max(x["ms_verify"], 1e-9) / 1e3, 1)}), flush=True)
