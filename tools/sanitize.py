#!/usr/bin/env python3
"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
~20 reference fixtures through every filter flavour -- tcgen05 int8 (two row
tiles), int8 single tile, fp4, the level-2 GEMM, the level-2 GEMM with the
head-overlap kernel (K3a), POPC -- which covers K1 build, K1b expand, K2,
K2b find/rescan/reduce, K3 verify, K3a head setup + GEMM, K4 small and radix
sorts; then 4 host threads joining at once (the concurrency the C ABI allows).
Every result is checked against the fixture, so a run under the sanitizer is
also a parity run.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize.py [flavour ...]
"""
import hashlib
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1711_07295_b200 import load_library  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

FLAVOURS = {
    "tcm": dict(SSJB_FILTER="tc", SSJB_TC_KIND="i8", SSJB_TCM="1", SSJB_L2GEMM="0", SSJB_HEAD="0"),
    "tc1": dict(SSJB_FILTER="tc", SSJB_TC_KIND="i8", SSJB_TCM="0", SSJB_L2GEMM="0", SSJB_HEAD="0"),
    "fp4": dict(SSJB_FILTER="tc", SSJB_TC_KIND="fp4", SSJB_L2GEMM="0", SSJB_HEAD="0"),
    "l2gemm": dict(SSJB_FILTER="tc", SSJB_TC_KIND="i8", SSJB_L2GEMM="1", SSJB_HEAD="0"),
    "head": dict(SSJB_FILTER="tc", SSJB_TC_KIND="i8", SSJB_L2GEMM="1", SSJB_HEAD="2", SSJB_HEAD_MIN_SIZE="3",
                 SSJB_HEAD_K="256", SSJB_HEAD_KIND="fp4", SSJB_ORDER_MIN_ROWS="1"),
    "head_i8": dict(SSJB_FILTER="tc", SSJB_TC_KIND="i8", SSJB_L2GEMM="1", SSJB_HEAD="2", SSJB_HEAD_MIN_SIZE="3",
                    SSJB_HEAD_K="128", SSJB_HEAD_KIND="i8", SSJB_ORDER_MIN_ROWS="1"),
    "popc": dict(SSJB_FILTER="popc", SSJB_L2GEMM="0", SSJB_HEAD="0"),
}


def main(names):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    arr = np.load(os.path.join(ROOT, "tests", "golden", "golden_pairs.npz"))
    lib = load_library()
    joins = [e for e in g["joins"] if e["pair_count"] > 0][:20]
    colls = {}

    def coll(name):
        if name not in colls:
            colls[name] = S.Collection.from_csr(lib, arr[f"coll/{name}/tokens"], arr[f"coll/{name}/offsets"])
        return colls[name]

    def run(e):
        o = S.default_options(lib)
        for k, v in e["options"].items():
            setattr(o, k, v)
        rep = S.join(coll(e["collection"]), o)
        ok = (len(rep.pairs) == e["pair_count"]
              and hashlib.sha256(rep.pairs.tobytes()).hexdigest() == e["pairs_sha256"]
              and all(rep.counters[k] == v for k, v in e["counters"].items()))
        return ok

    bad = 0
    for name in names or list(FLAVOURS):
        os.environ.update(FLAVOURS[name])
        res = [run(e) for e in joins]
        bad += res.count(False)
        print(f"{name}: {sum(res)}/{len(res)} fixtures exact", flush=True)
    os.environ.update(FLAVOURS["tcm"])
    with ThreadPoolExecutor(max_workers=4) as pool:
        res = list(pool.map(run, joins))
    bad += res.count(False)
    print(f"4 threads: {sum(res)}/{len(res)} fixtures exact", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main(sys.argv[1:])
