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


# ---- heavy-tailed collections (BASELINE configs 3-5) ------------------------
#
# The reference generator only draws Poisson sizes; KOSARAK/ORKUT/AOL have
# heavy-tailed lengths (PAPER.md table "Collections used in experiments"), so
# these shapes are drawn here with a seeded numpy Generator (deterministic for
# a given numpy version) and canonicalised through the library's loader
# (ssjb_collection_from_csr = reference id-file path, src/collection.cpp:97-137).
# Tokens follow a bounded Zipf law (continuous inverse CDF, rank 1 the most
# frequent); rank r is written as token id universe - r so frequent tokens get
# large ids, as the reference's rarest-first renumbering would
# (src/collection.cpp:68-82).  Duplicates inside a record collapse when the
# loader canonicalises it, so sizes shrink slightly at the heavy Zipf head.

def zipf_ranks(rng, count: int, universe: int, exponent: float) -> np.ndarray:
    """`count` ranks in [1, universe] with P(r) ~ r^-exponent (inverse CDF of
    the continuous law over [1, universe+1), floored)."""
    u = rng.random(count)
    if abs(exponent - 1.0) < 1e-12:
        r = np.exp(u * np.log(universe + 1.0))
    else:
        a = 1.0 - exponent
        r = (u * ((universe + 1.0) ** a - 1.0) + 1.0) ** (1.0 / a)
    return np.minimum(np.floor(r), universe).astype(np.int64)


def lognormal_sizes(rng, n: int, median: float, mean: float, max_size: int) -> np.ndarray:
    """Sizes with the given median and (pre-clip) mean, clipped to [1, max_size]."""
    mu = np.log(median)
    sigma = np.sqrt(2.0 * np.log(mean / median))
    s = np.rint(rng.lognormal(mu, sigma, n))
    return np.clip(s, 1, max_size).astype(np.int64)


def from_sizes(lib, rng, sizes: np.ndarray, universe: int, exponent: float) -> S.Collection:
    offsets = np.zeros(len(sizes) + 1, dtype=np.uint64)
    np.cumsum(sizes, out=offsets[1:])
    total = int(offsets[-1])
    tokens = np.empty(total, dtype=np.uint32)
    chunk = 1 << 26
    for a in range(0, total, chunk):
        b = min(total, a + chunk)
        tokens[a:b] = (universe - zipf_ranks(rng, b - a, universe, exponent)).astype(np.uint32)
    return S.Collection.from_csr(lib, tokens, offsets)


def c3(lib, num_sets: int = 606770, seed: int = 3) -> S.Collection:
    """KOSARAK-shaped: 606,770 sets, lognormal sizes (median 5, mean 11.93,
    max 2,498), Zipf tokens over 41,275 (PAPER.md: kosarak)."""
    rng = np.random.default_rng(seed)
    sizes = lognormal_sizes(rng, num_sets, 5, 11.93, 2498)
    return from_sizes(lib, rng, sizes, 41275, 1.0)


def c4(lib, num_sets: int = 2732271, seed: int = 4) -> S.Collection:
    """ORKUT-shaped: 2,732,271 sets, lognormal sizes (median 29, max 40,425),
    Zipf tokens over 8,730,857 (PAPER.md: orkut).  The pre-dedup mean 155
    lands the canonical mean at ~120 (orkut: 119.67) once Zipf-head repeats
    collapse."""
    rng = np.random.default_rng(seed)
    sizes = lognormal_sizes(rng, num_sets, 29, 155, 40425)
    return from_sizes(lib, rng, sizes, 8730857, 1.0)


C5_EXPONENT = 0.75


def c5(lib, num_sets: int = 10_000_000, seed: int = 5) -> S.Collection:
    """AOL/SPOT-shaped: 10M sets, sizes 1 + Poisson(2.01) (mean 3.01, median 3)
    with a 0.1% lognormal tail up to 245, Zipf tokens over 3,873,246.  The
    exponent (C5_EXPONENT) is flattened from 1 so the tau = 0.8 output stays
    ~1e8 pairs instead of the ~8e9 an exponent of 1 implies."""
    rng = np.random.default_rng(seed)
    sizes = 1 + rng.poisson(2.01, num_sets)
    tail = rng.random(num_sets) < 0.001
    sizes[tail] = lognormal_sizes(rng, int(tail.sum()), 8, 20, 245)
    return from_sizes(lib, rng, sizes.astype(np.int64), 3873246, C5_EXPONENT)


def c3_options(lib, **kw):
    """C3 join: Jaccard 1/2, Bitmap-Next, b = 64, cutoff OFF."""
    return S.par_bitmap_options(lib, threshold=(1, 2), method=capi.SSJ_BITMAP_NEXT, bits=64,
                                cutoff_mode=capi.SSJ_CUTOFF_OFF, **kw)


def c4_options(lib, bits=64, **kw):
    """C4 join: Jaccard 7/10, Bitmap-Xor, b = 64 (what auto resolves to) or 128."""
    return S.par_bitmap_options(lib, threshold=(7, 10), method=capi.SSJ_BITMAP_XOR, bits=bits,
                                cutoff_mode=capi.SSJ_CUTOFF_OFF, **kw)


def c5_options(lib, **kw):
    """C5 join: Jaccard 4/5, Bitmap-Xor, b = 256, cutoff OFF."""
    return S.par_bitmap_options(lib, threshold=(4, 5), method=capi.SSJ_BITMAP_XOR, bits=256,
                                cutoff_mode=capi.SSJ_CUTOFF_OFF, **kw)


def window_pairs(offsets: np.ndarray, p: int, q: int) -> int:
    """Sum over rows of the length-filter window i - j0(i) (the reference's
    `candidates` before saturation, src/parallel_join.cpp:65-73)."""
    sizes = np.diff(offsets.astype(np.int64))
    min_size = -((-p * sizes) // q)  # ceil(p*|r|/q)
    j0 = np.searchsorted(sizes, min_size, side="left")
    return int((np.arange(len(sizes)) - np.minimum(j0, np.arange(len(sizes)))).sum())
