#!/usr/bin/env python3
"""Workload for compute-sanitizer over the prefix-filter engine (round 2,
csrc/prefix_join.cuh) and the CTA-per-record sketch build: a spread of
golden_prefix fixtures (every algorithm, similarity function and bitmap
placement, the edge collections, forced result overflow) and a heavy-tailed
sketch build (lane-group / warp / CTA tiers), each checked against its
reference fixture or the oracle, so a sanitizer run is also a parity run.

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_prefix.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (checker)
from paper_1711_07295_b200 import capi, load_library  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    lib = load_library()
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "golden_prefix.json")))["cases"]
    arr = np.load(os.path.join(ROOT, "tests", "golden", "golden_prefix.npz"))
    colls, n = {}, 0
    for k, c in enumerate(cases):
        if k % 23 and c["collection"] not in ("edge", "one", "empty"):
            continue
        if c["collection"] in ("edge", "one", "empty") and k % 3:
            continue
        name = c["collection"]
        if name not in colls:
            colls[name] = S.Collection.from_csr(lib, arr[f"coll/{name}/tokens"], arr[f"coll/{name}/offsets"])
        o = S.default_options(lib)
        for f, v in c["options"].items():
            setattr(o, f, v)
        if k % 2:
            os.environ["SSJB_PREFIX_RESULT_CAP"] = "64"
        rep = S.join(colls[name], o)
        os.environ.pop("SSJB_PREFIX_RESULT_CAP", None)
        assert rep.counters == c["counters"] and sha(rep.pairs) == c["pairs_sha256"], c["id"]
        n += 1
    rng = np.random.default_rng(5)
    sizes = np.minimum(np.maximum(1, rng.lognormal(np.log(40), 1.4, 1500).astype(np.int64)), 9000)
    recs = [np.unique(rng.integers(0, 100000, int(z))).tolist() for z in sizes]
    coll = S.Collection.from_records(lib, recs)
    t, off = coll.csr()
    for method in (capi.SSJ_BITMAP_SET, capi.SSJ_BITMAP_XOR):
        for bits in (64, 256):
            assert (S.build_bitmaps(coll, method, bits, 1) == O.build_bitmaps(t, off, method, bits, 1)).all()
    print(f"sanitize_prefix ok: {n} prefix-filter joins, 4 heavy-tail sketch stores")


if __name__ == "__main__":
    main()
