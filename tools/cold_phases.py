#!/usr/bin/env python3
"""Cold vs warm ssj_join on C4: the first join of the process on a fresh
collection, a second fresh collection (library warm, collection cold), then
warm joins -- wall time and the library's phase times for each."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

lib = pkg.load_library()
base = D.c4(lib)
t, o = base.csr()
for label in ("process-cold", "collection-cold", "warm", "warm"):
    c = S.Collection.from_csr(lib, t, o) if label.endswith("cold") else base
    t0 = time.perf_counter()
    r = S.join(c, D.c4_options(lib))
    wall = time.perf_counter() - t0
    x = r.extra
    print(json.dumps({"run": label, "wall_s": round(wall, 3), "timings": r.timings,
                      "ms": {k[3:]: round(x[k], 2) for k in x if k.startswith("ms_")},
                      "h2d": x.get("h2d_bytes"), "d2h": x.get("d2h_bytes")}), flush=True)
    del r
    if label.endswith("cold"):
        c.close()
