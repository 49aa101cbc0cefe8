#!/usr/bin/env python3
"""Full-size prefix-filter joins from the UNMODIFIED reference
(oracle/_ref/libssjoin_ref.so): ALLPAIRS / PPJOIN / PPJOIN+ / GROUPJOIN /
ADAPTJOIN with the Bitmap Filter (filter3, and filter2 for some) on the
BASELINE-shaped C1 (tau 0.9), C2 (tau 0.8), C3 (tau 0.5) and C4 (tau 0.7,
ALLPAIRS, PPJOIN and GROUPJOIN: ~9-10 min each) collections
(paper_1711_07295_b200.datasets).  One process per join (single-threaded, as
the reference runs these algorithms), several in parallel; each records the
collection sha256, the options, the full pair list's count and sha256, the
nine counters and the reference's own timings.  Output: prefix_large.jsonl.

    python tests/golden/make_golden_prefix_large.py      # ~15 min on 8 cores
"""
import concurrent.futures as cf
import hashlib
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "prefix_large.jsonl")
TAU = {"c1": (9, 10), "c2": (4, 5), "c3": (1, 2), "c4": (7, 10)}
JOBS = ([("c1", a, "f3") for a in (1, 2, 3, 4, 5)] + [("c1", a, "f2") for a in (1, 2, 3)] +
        [("c2", a, "f3") for a in (1, 2, 3, 4, 5)] + [("c2", 1, "f2"), ("c2", 3, "f2")] +
        [("c3", a, "f3") for a in (1, 2, 3, 4)] + [("c3", 2, "f2")] +
        [("c4", a, "f3") for a in (1, 2, 4)])


def one(name, algo, bl):
    sys.path.insert(0, ROOT)
    import numpy as np
    from oracle import oracle as O
    from paper_1711_07295_b200 import capi, datasets as D
    from paper_1711_07295_b200 import ssjoin as S
    ref = O.ref_lib()
    c = getattr(D, name)(ref)
    t, o = c.csr()
    kw = {"f3": dict(bitmap_enabled=1), "f2": dict(bitmap_enabled=1, placement=capi.SSJ_PLACEMENT_FILTER2)}[bl]
    opts = S.default_options(ref, algorithm=algo, threshold=TAU[name], **kw)
    t0 = time.perf_counter()
    r = S.join(c, opts)
    dt = time.perf_counter() - t0
    return dict(config=name, algo=algo, bitmap=bl, join_s=round(dt, 3), pair_count=int(len(r.pairs)),
                pairs_sha256=hashlib.sha256(np.ascontiguousarray(r.pairs).tobytes()).hexdigest(),
                collection_sha256=hashlib.sha256(np.ascontiguousarray(t).tobytes() +
                                                 np.ascontiguousarray(o).tobytes()).hexdigest(),
                options={k: getattr(opts, k) for k, _ in capi.JoinOptions._fields_},
                counters=r.counters, timings=r.timings)


def main():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True)
    with cf.ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        res = list(ex.map(one, *zip(*JOBS)))
    with open(OUT, "w") as f:
        for d in res:
            f.write(json.dumps(d) + "\n")
    print(f"{len(res)} joins -> {OUT}")


if __name__ == "__main__":
    main()
