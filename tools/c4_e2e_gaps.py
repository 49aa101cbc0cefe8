#!/usr/bin/env python3
"""Where the C4 END-TO-END join (ssj_join on a host collection, as bench.py's
`e2e`) spends its time: host phase trace (SSJB_HOST_TIMING=2, stderr), wall
time and device phase sums per join."""
import json
import os
import sys
import time

os.environ.setdefault("SSJB_HOST_TIMING", "2")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

lib = pkg.load_library()
c = D.c4(lib)
o = D.c4_options(lib)
pass
for k in range(6):
    print(f"---- join {k}", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    r = S.join(c, o)
    wall = (time.perf_counter() - t0) * 1e3
    x = r.extra
    dev = sum(x[k2] for k2 in x if k2.startswith("ms_") and k2 not in ("ms_merge",))
    print(json.dumps({"join": k, "wall_ms": round(wall, 2), "device_phase_ms": round(dev, 2),
                      "ms": {k2[3:]: round(x[k2], 2) for k2 in x if k2.startswith("ms_")}}), flush=True)
    r.pairs = None
    del r
