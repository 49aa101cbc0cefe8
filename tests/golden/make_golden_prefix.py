#!/usr/bin/env python3
"""Regenerates tests/golden/golden_prefix.{json,npz}: the reference's
prefix-filter joins -- ALLPAIRS, PPJOIN, PPJOIN+ (src/join.cpp:132-189),
GROUPJOIN (:197-329), ADAPTJOIN (:331-420) -- with and without the Bitmap
Filter (filter3 default placement and filter2 inside the candidate loop), for
every similarity function, from the UNMODIFIED reference engine
(oracle/_ref/libssjoin_ref.so, built by `make -C oracle` from /root/reference
sources).  Each case records the full pair list and all nine counters, which
are algorithm-specific (prefix_index.cpp:53-148 counts per probe walk).

The collections follow the reference's own join tests
(tests/test_joins.cpp:62-112: random_collection(300, 6, 30 | 400, seed 11 | 12)
at its Jaccard threshold grid and Cosine / Dice / Overlap thresholds), plus
Zipf, wide-record, duplicate-heavy (GroupJoin groups) and edge-case
collections.

    python tests/golden/make_golden_prefix.py

Runs only in the build container; the GPU box reads the committed fixtures.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1711_07295_b200 import capi  # noqa: E402
from paper_1711_07295_b200 import ssjoin as S  # noqa: E402

REF_SO = os.path.join(ROOT, "oracle", "_ref", "libssjoin_ref.so")
OUT_DIR = os.path.dirname(os.path.abspath(__file__))

OV, JAC, COS, DICE = capi.SSJ_SIM_OVERLAP, capi.SSJ_SIM_JACCARD, capi.SSJ_SIM_COSINE, capi.SSJ_SIM_DICE
ALGOS = (capi.SSJ_ALGO_ALLPAIRS, capi.SSJ_ALGO_PPJOIN, capi.SSJ_ALGO_PPJOIN_PLUS, capi.SSJ_ALGO_GROUPJOIN,
         capi.SSJ_ALGO_ADAPTJOIN)

# bitmap variants: (label, option overrides)
BITMAPS = (
    ("off", dict(bitmap_enabled=0)),
    ("f3", dict(bitmap_enabled=1)),                                      # Combined, auto width, AUTO cutoff
    ("f2", dict(bitmap_enabled=1, placement=capi.SSJ_PLACEMENT_FILTER2)),
    ("f3-xor128-mult-cut", dict(bitmap_enabled=1, bitmap_method=capi.SSJ_BITMAP_XOR, bitmap_bits=128,
                                bitmap_hash=capi.SSJ_HASH_MULT, cutoff_mode=capi.SSJ_CUTOFF_EXPLICIT,
                                cutoff_value=9)),
    ("f2-next-off", dict(bitmap_enabled=1, bitmap_method=capi.SSJ_BITMAP_NEXT, cutoff_mode=capi.SSJ_CUTOFF_OFF,
                         placement=capi.SSJ_PLACEMENT_FILTER2)),
)


def main() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True)
    ref = capi.bind(C.CDLL(REF_SO))
    store, cases, colls = {}, [], {}

    def keep(name, coll):
        t, o = coll.csr()
        store[f"coll/{name}/tokens"] = t
        store[f"coll/{name}/offsets"] = o
        colls[name] = coll

    keep("r11", S.Collection.generate(ref, 300, 6, 30, 11))      # test_joins.cpp:66-68
    keep("r12", S.Collection.generate(ref, 300, 6, 400, 12))
    keep("z900", S.Collection.generate(ref, 900, 12, 500, 31, capi.SSJ_DIST_ZIPF))
    keep("w200", S.Collection.generate(ref, 200, 60, 300, 32))
    rng = np.random.default_rng(33)
    base = [sorted(set(rng.integers(0, 40, int(rng.integers(1, 9))).tolist())) for _ in range(60)]
    dup = [base[int(rng.integers(0, 60))] for _ in range(500)]
    dup += [sorted(set(b + [int(rng.integers(40, 80))])) for b in base[:40]]
    keep("dups", S.Collection.from_records(ref, dup))           # many GroupJoin groups of size > 1
    keep("edge", S.Collection.from_records(ref, [[]] * 3 + [[1, 2, 3], [1, 2, 3], [2, 3], [4], [1, 2, 3, 4],
                                                            [7, 8, 9]] + [[7, 8, 9]] * 4))
    keep("one", S.Collection.from_records(ref, [[1, 2, 3]]))
    keep("empty", S.Collection.from_records(ref, []))

    def run(coll, sim, tau, algo, blabel, bopts, extra=None, label=""):
        kw = dict(algorithm=algo, similarity=sim, threshold=tau, **bopts)
        if extra:
            kw.update(extra)
        opts = S.default_options(ref, **kw)
        rep = S.join(colls[coll], opts)
        cid = f"p{len(cases):04d}"
        if len(rep.pairs) <= 2000:  # larger lists are pinned by their sha256
            store[f"pairs/{cid}"] = rep.pairs
        rec = {k: getattr(opts, k) for k, _ in capi.JoinOptions._fields_}
        cases.append(dict(id=cid, collection=coll, options=rec, label=f"{label} {blabel}".strip(),
                          counters=rep.counters, pair_count=int(len(rep.pairs)),
                          pairs_sha256=hashlib.sha256(np.ascontiguousarray(rep.pairs).tobytes()).hexdigest()))

    jac = [(1, 2), (3, 5), (7, 10), (4, 5), (9, 10), (1, 1)]
    other = [(COS, (1, 2)), (COS, (7, 10)), (COS, (9, 10)), (DICE, (1, 2)), (DICE, (7, 10)), (DICE, (9, 10)),
             (OV, (3, 1)), (OV, (5, 1))]
    for coll in ("r11", "r12", "z900", "dups"):
        for tau in jac:
            for algo in ALGOS:
                for bl, bo in BITMAPS:
                    run(coll, JAC, tau, algo, bl, bo)
        for sim, tau in other:
            for algo in ALGOS:
                for bl, bo in BITMAPS[:3]:
                    run(coll, sim, tau, algo, bl, bo)
    for coll in ("w200", "edge", "one", "empty"):
        for sim, tau in ((JAC, (1, 2)), (JAC, (4, 5)), (COS, (7, 10)), (DICE, (3, 5)), (OV, (2, 1))):
            for algo in ALGOS:
                for bl, bo in BITMAPS[:3]:
                    run(coll, sim, tau, algo, bl, bo)
    # PPJoin+ partition depth and AdaptJoin prefix-extension cap
    for coll in ("r11", "z900", "w200"):
        for tau in ((1, 2), (7, 10)):
            for depth in (0, 1, 4, 9):
                run(coll, JAC, tau, capi.SSJ_ALGO_PPJOIN_PLUS, "off", BITMAPS[0][1], dict(suffix_depth=depth),
                    f"suffix_depth={depth}")
            for ell in (0, 1, 2, 5, 8):
                for bl, bo in BITMAPS[:2]:
                    run(coll, JAC, tau, capi.SSJ_ALGO_ADAPTJOIN, bl, bo, dict(ell_max=ell), f"ell_max={ell}")

    np.savez_compressed(os.path.join(OUT_DIR, "golden_prefix.npz"), **store)
    with open(os.path.join(OUT_DIR, "golden_prefix.json"), "w") as f:
        json.dump({"source": "reference ssj_join(ALLPAIRS..ADAPTJOIN) via oracle/_ref/libssjoin_ref.so",
                   "cases": cases}, f, indent=0)
    print(f"{len(cases)} prefix-filter cases, {sum(c['pair_count'] for c in cases)} pairs")


if __name__ == "__main__":
    main()
