#!/usr/bin/env python3
"""Full-size golden results of the BASELINE configs, computed by the
UNMODIFIED reference (oracle/_ref/libssjoin_ref.so, ssj_join PAR_BITMAP with
8 workers) in the build container.  Appends one JSON line per case to
tests/golden/large.jsonl (pairs inline when <= 50,000, else their sha256);
existing cases are skipped so the script can be resumed.

    python tests/golden/make_golden_large.py [case-prefix ...]
"""
from __future__ import annotations

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


def main(prefixes):
    ref = capi.bind(C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libssjoin_ref.so")))
    done = set()
    if os.path.exists(OUT):
        for line in open(OUT):
            done.add(json.loads(line)["case"])
    cases = [("C1", lambda: D.c1(ref), (9, 10), 64),
             ("C3", lambda: D.c3(ref), (1, 2), 64)]
    for bits in (128, 256):
        for tau in reversed(D.C2_TAUS):
            cases.append((f"C2_b{bits}_{tau[0]}_{tau[1]}", None, tau, bits))
    c2 = None
    for name, mk, tau, bits in cases:
        if name in done or (prefixes and not any(name.startswith(p) for p in prefixes)):
            continue
        if mk is not None:
            coll = mk()
        else:
            if c2 is None:
                c2 = D.c2(ref)
            coll = c2
        method = capi.SSJ_BITMAP_NEXT if name == "C3" else capi.SSJ_BITMAP_XOR
        opts = S.par_bitmap_options(ref, threshold=tau, method=method, bits=bits,
                                    cutoff_mode=capi.SSJ_CUTOFF_OFF, workers=os.cpu_count() or 8)
        t, o = coll.csr()
        t0 = time.time()
        rep = S.join(coll, opts)
        wall = time.time() - t0
        entry = dict(case=name, tau=list(tau), bits=bits, method=method, counters=rep.counters,
                     collection_sha256=hashlib.sha256(t.tobytes() + o.tobytes()).hexdigest(),
                     saturated_records=rep.saturated_records, pair_count=int(len(rep.pairs)),
                     pairs_sha256=hashlib.sha256(rep.pairs.tobytes()).hexdigest(),
                     ref_total_s=rep.timings["total_s"], ref_wall_s=wall, workers=opts.workers)
        if len(rep.pairs) <= 50000:
            entry["pairs"] = rep.pairs.view(np.uint32).reshape(-1, 4)[:, [0, 1, 2]].tolist()
        with open(OUT, "a") as f:
            f.write(json.dumps(entry) + "\n")
        print(name, rep.counters["candidates"], len(rep.pairs), f"{wall:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
