#!/usr/bin/env python3
"""C4 end-to-end ssj_join (host collection, streamed ingest) for several
SSJB_STREAM_CHUNKS settings: wall time per warm join, and the pair list
checked against the reference's (tests/golden/large.jsonl C4_exact)."""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_07295_b200 as pkg  # noqa: E402
from paper_1711_07295_b200 import datasets as D  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

want = next(d for d in map(json.loads, open(os.path.join(ROOT, "tests", "golden", "large.jsonl")))
            if d.get("case") == "C4_exact")
lib = pkg.load_library()
c = D.c4(lib)
o = D.c4_options(lib)
for chunks in sys.argv[1:] or ["2", "4", "8"]:
    os.environ["SSJB_STREAM_CHUNKS"] = chunks
    walls = []
    for k in range(5):
        t0 = time.perf_counter()
        r = S.join(c, o)
        walls.append((time.perf_counter() - t0) * 1e3)
        if k == 4:
            ok = len(r.pairs) == want["pair_count"] and \
                hashlib.sha256(np.ascontiguousarray(r.pairs).tobytes()).hexdigest() == want["pairs_sha256"]
        r.pairs = None
        del r
    print(json.dumps({"chunks": int(chunks), "wall_ms": [round(w, 1) for w in walls], "pairs_ok": ok}), flush=True)
