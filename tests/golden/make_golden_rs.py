#!/usr/bin/env python3
"""Regenerates tests/golden/golden_rs.{json,npz}: NAIVE joins with every
similarity function, self-joins and RS-joins (two collections), from the
UNMODIFIED reference engine (oracle/_ref/libssjoin_ref.so, built by
`make -C oracle` from /root/reference sources).

The reference supports RS-joins only through the naive algorithm
(src/capi.cpp:225-232 -> src/join.cpp:110-121) and the naive join accepts
Overlap / Jaccard / Cosine / Dice thresholds (src/similarity.cpp:18-27,93-115).

    python tests/golden/make_golden_rs.py

Runs only in the build container; the GPU box reads the committed fixtures.
"""
from __future__ import annotations

import ctypes as C
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


def main() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"], check=True)
    ref = capi.bind(C.CDLL(REF_SO))
    store, cases, colls = {}, [], {}

    def keep(name, coll):
        t, o = coll.csr()
        store[f"coll/{name}/tokens"] = t
        store[f"coll/{name}/offsets"] = o
        colls[name] = coll

    keep("u300", S.Collection.generate(ref, 300, 8, 60, 21))
    keep("u250", S.Collection.generate(ref, 250, 8, 60, 22))
    keep("z700", S.Collection.generate(ref, 700, 14, 300, 23, capi.SSJ_DIST_ZIPF))
    keep("z400", S.Collection.generate(ref, 400, 30, 500, 24, capi.SSJ_DIST_ZIPF))
    keep("w150", S.Collection.generate(ref, 150, 90, 2000, 25))
    keep("edge", S.Collection.from_records(ref, [[]] * 3 + [[1, 2, 3], [1, 2, 3], [2, 3], [4]]))
    keep("edge2", S.Collection.from_records(ref, [[], [1, 2], [1, 2, 3], [9]]))
    keep("one", S.Collection.from_records(ref, [[1, 2, 3]]))
    keep("empty", S.Collection.from_records(ref, []))

    sims = [(JAC, (1, 2)), (JAC, (7, 10)), (JAC, (1, 1)), (DICE, (7, 10)), (DICE, (9, 10)),
            (COS, (7, 10)), (COS, (4, 5)), (COS, (1, 3)), (OV, (3, 1)), (OV, (6, 1))]

    def run(r, s, sim, tau, label):
        opts = S.default_options(ref, algorithm=capi.SSJ_ALGO_NAIVE, similarity=sim, threshold=tau)
        rep = S.join(colls[r], opts, colls[s] if s else None)
        cid = f"n{len(cases):03d}"
        store[f"pairs/{cid}"] = rep.pairs
        cases.append(dict(id=cid, r=r, s=s, similarity=sim, threshold=list(tau), label=label,
                          counters=rep.counters, saturated_records=rep.saturated_records,
                          pair_count=int(len(rep.pairs))))

    for sim, tau in sims:
        run("u300", "u250", sim, tau, "RS uniform")
        run("z700", "z400", sim, tau, "RS zipf")
        run("u300", None, sim, tau, "self")
    for sim, tau in ((JAC, (1, 2)), (COS, (7, 10)), (OV, (1, 1)), (DICE, (1, 2))):
        run("w150", "z400", sim, tau, "RS wide x zipf")
        run("edge", "edge2", sim, tau, "RS empty records")
        run("edge2", "edge", sim, tau, "RS empty records swapped")
        run("one", "edge", sim, tau, "RS single record")
        run("empty", "u250", sim, tau, "RS empty R")
        run("u250", "empty", sim, tau, "RS empty S")
        run("z700", "z700", sim, tau, "RS collection with itself")
        run("edge", None, sim, tau, "self empty records")

    np.savez_compressed(os.path.join(OUT_DIR, "golden_rs.npz"), **store)
    with open(os.path.join(OUT_DIR, "golden_rs.json"), "w") as f:
        json.dump({"source": "reference ssj_join(NAIVE) via oracle/_ref/libssjoin_ref.so",
                   "cases": cases}, f, indent=1)
    print(f"{len(cases)} naive cases, {sum(c['pair_count'] for c in cases)} pairs")


if __name__ == "__main__":
    main()
