"""Synthetic workloads of BASELINE.json's configs (host-side data preparation).

Every collection is built through the reference-compatible generator
(``ssj_collection_generate``, bit-identical to reference
src/collection.cpp:193-254) plus, where the config needs non-trivial output,
deterministic planted near-duplicates; the result is canonicalised through
the library's own loader, so any engine given the same CSR assigns the same
record ids (reference src/collection.cpp:44-54).

  C1  uniform, 100K sets, mean 10, universe 220, seed 1       (the paper's `uniform`)
  C2  DBLP-shaped: Zipf tokens over 4,000, Poisson mean 86, 100K sets
      (99,000 generated + 1,000 planted copies with 1..8 token edits)
"""
from __future__ import annotations

import numpy as np

from . import capi
from . import ssjoin as S

C2_TAUS = ((1, 2), (3, 5), (7, 10), (3, 4), (4, 5), (17, 20), (9, 10), (19, 20))


def c1(lib) -> S.Collection:
    return S.Collection.generate(lib, 100000, 10, 220, 1, capi.SSJ_DIST_UNIFORM)


def planted(lib, base: S.Collection, copies: int, max_edits: int, universe: int, seed: int) -> S.Collection:
    """base + `copies` near-duplicates: a random base record with k in
    [1, max_edits] tokens replaced by uniform draws over the universe."""
    t, o = base.csr()
    rng = np.random.default_rng(seed)
    n = len(o) - 1
    src = rng.integers(0, n, size=copies)
    edits = rng.integers(1, max_edits + 1, size=copies)
    recs = [t[int(o[r]):int(o[r + 1])] for r in range(n)]
    for s, k in zip(src.tolist(), edits.tolist()):
        rec = recs[s].copy()
        if len(rec):
            pos = rng.choice(len(rec), size=min(k, len(rec)), replace=False)
            rec[pos] = rng.integers(0, universe, size=len(pos), dtype=np.uint32)
        recs.append(rec)
    lens = np.fromiter((len(r) for r in recs), dtype=np.uint64, count=len(recs))
    offsets = np.zeros(len(recs) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offsets[1:])
    tokens = np.concatenate(recs).astype(np.uint32)
    return S.Collection.from_csr(lib, tokens, offsets)


def c2(lib, num_sets: int = 100000, planted_frac: float = 0.01, seed: int = 1) -> S.Collection:
    copies = int(round(num_sets * planted_frac))
    base = S.Collection.generate(lib, num_sets - copies, 86, 4000, seed, capi.SSJ_DIST_ZIPF)
    return planted(lib, base, copies, 8, 4000, seed + 1000)


def c2_options(lib, tau, bits=128, **kw):
    """C2 join: Jaccard tau, Bitmap-Xor, b bits, cutoff OFF (the paper's GPU setting)."""
    return S.par_bitmap_options(lib, threshold=tau, method=capi.SSJ_BITMAP_XOR, bits=bits,
                                cutoff_mode=capi.SSJ_CUTOFF_OFF, **kw)


def c1_options(lib, **kw):
    return S.par_bitmap_options(lib, threshold=(9, 10), method=capi.SSJ_BITMAP_XOR, bits=64,
                                cutoff_mode=capi.SSJ_CUTOFF_OFF, **kw)
