"""NAIVE joins with every similarity function, self-joins and RS-joins (two
collections) -- reference src/join.cpp:91-126 via src/capi.cpp:225-232.

Fixtures: tests/golden/golden_rs.{json,npz}, produced by the unmodified
reference (tests/golden/make_golden_rs.py).  CPU tests pin the oracle to
them; `-m gpu` tests run the B200 library through ssj_join and compare
pairs, overlaps and counters bit-exactly."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from paper_1711_07295_b200 import capi
from paper_1711_07295_b200 import ssjoin as S

COUNTER_KEYS = ("candidates", "pruned_length", "pruned_positional", "pruned_suffix", "pruned_bitmap",
                "bitmap_tested", "filter_evaluations", "verified", "matched")


@pytest.fixture(scope="module")
def rs_golden():
    with open(os.path.join(GOLDEN_DIR, "golden_rs.json")) as f:
        cases = json.load(f)["cases"]
    return cases, np.load(os.path.join(GOLDEN_DIR, "golden_rs.npz"))


def _csr(arrs, name):
    return arrs[f"coll/{name}/tokens"], arrs[f"coll/{name}/offsets"]


def test_oracle_required_overlap_all_similarities(oracle):
    # reference tests/test_similarity.cpp:102 and the closed forms of src/similarity.cpp:93-111
    assert oracle.required_overlap_sim(1, 3, 5, 7, 6) == 5          # Jaccard 3/5, 7, 6
    assert oracle.required_overlap_sim(0, 4, 1, 10, 3) == 4         # Overlap 4
    assert oracle.required_overlap_sim(3, 1, 2, 10, 10) == 5        # Dice 1/2: ceil(20/4)
    assert oracle.required_overlap_sim(2, 1, 2, 9, 4) == 3          # Cosine 1/2: ceil(sqrt(36)/2)
    assert oracle.required_overlap_sim(2, 7, 10, 10, 10) == 7       # Cosine 7/10: 0.7*10
    assert oracle.required_overlap_sim(2, 1, 3, 1, 1) == 1          # clamp to 1
    assert oracle.required_overlap_sim(1, 1, 2, 0, 0) == 1


def test_oracle_matches_reference_naive_fixtures(oracle, rs_golden):
    cases, arrs = rs_golden
    for e in cases:
        rt, ro = _csr(arrs, e["r"])
        p, q = e["threshold"]
        if e["s"] is None:
            pairs, cnt = oracle.naive_join_sim(rt, ro, e["similarity"], p, q)
        else:
            st, so = _csr(arrs, e["s"])
            pairs, cnt = oracle.naive_join_sim(rt, ro, e["similarity"], p, q, st, so)
        want = arrs[f"pairs/{e['id']}"]
        assert len(pairs) == e["pair_count"], e
        assert (pairs == want).all(), e
        for k in ("candidates", "verified", "matched"):
            assert cnt[k] == e["counters"][k], (e, k)


def test_rs_join_rejects_non_naive_algorithms(lib):
    r = S.Collection.from_records(lib, [[1, 2, 3], [2, 3]])
    s = S.Collection.from_records(lib, [[1, 2, 3]])
    opts = S.par_bitmap_options(lib, threshold=(1, 2))
    with pytest.raises(S.SsjError) as ei:
        S.join(r, opts, s)
    assert ei.value.status == capi.SSJ_ERROR_INVALID_ARGUMENT
    assert "naive" in str(ei.value)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["filtered", "brute"])
def test_gpu_naive_joins_match_reference(lib, rs_golden, mode, monkeypatch):
    """Every reference NAIVE fixture; RS-joins through the filtered R x S path
    (length window + Xor sketch bound, forced on) and through the brute-force
    merge of every pair."""
    monkeypatch.setenv("SSJB_RS_FILTER", "2" if mode == "filtered" else "0")
    cases, arrs = rs_golden
    colls = {}

    def get(name):
        if name not in colls:
            colls[name] = S.Collection.from_csr(lib, *_csr(arrs, name))
        return colls[name]

    for e in cases:
        opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE, similarity=e["similarity"],
                                 threshold=tuple(e["threshold"]))
        rep = S.join(get(e["r"]), opts, get(e["s"]) if e["s"] else None)
        want = arrs[f"pairs/{e['id']}"]
        assert len(rep.pairs) == e["pair_count"], e
        assert rep.pairs.tobytes() == want.tobytes(), e
        for k in COUNTER_KEYS:
            assert rep.counters[k] == e["counters"][k], (e, k)
        assert rep.saturated_records == e["saturated_records"]


@pytest.mark.gpu
def test_gpu_filtered_rs_join_merges_far_fewer_pairs(lib, monkeypatch):
    """30,000 x 30,000 Zipf-token records at Jaccard 0.6: the filtered RS path
    returns the brute-force pair list and NAIVE's counters while merging at
    least 100x fewer pairs (ssjb_stats.survivors)."""
    r = S.Collection.generate(lib, 30000, 10, 1000, 41, capi.SSJ_DIST_ZIPF, 1.0)
    s = S.Collection.generate(lib, 30000, 10, 1000, 42, capi.SSJ_DIST_ZIPF, 1.0)
    opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE, threshold=(3, 5))
    monkeypatch.setenv("SSJB_RS_FILTER", "0")
    brute = S.join(r, opts, s)
    monkeypatch.setenv("SSJB_RS_FILTER", "2")
    filt = S.join(r, opts, s)
    assert brute.pairs.tobytes() == filt.pairs.tobytes()
    assert filt.counters == brute.counters
    assert filt.counters["candidates"] == 30000 * 30000 == filt.counters["verified"]
    assert filt.extra["survivors"] * 100 <= 30000 * 30000, filt.extra
    print(f"filtered RS: {len(filt.pairs)} pairs, {filt.extra['survivors']} merges of {30000 * 30000}")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["filtered", "brute"])
def test_gpu_rs_join_batches_and_result_overflow(lib, oracle, monkeypatch, mode):
    """Small launch ranges and a tiny result buffer force many runs and
    overflow redos; the concatenated runs must still be the canonical list."""
    r = S.Collection.generate(lib, 900, 10, 80, 31)
    s = S.Collection.generate(lib, 700, 10, 80, 32)
    rt, ro = r.csr()
    st, so = s.csr()
    want, cnt = oracle.naive_join_sim(rt, ro, capi.SSJ_SIM_JACCARD, 1, 3, st, so)
    opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE, threshold=(1, 3))
    base = S.join(r, opts, s)
    assert (base.pairs == want).all() and base.counters["matched"] == cnt["matched"]
    monkeypatch.setenv("SSJB_RS_BATCH", "50000")
    monkeypatch.setenv("SSJB_RESULT_CAP", "1024")
    monkeypatch.setenv("SSJB_RS_FILTER", "2" if mode == "filtered" else "0")
    rep = S.join(r, opts, s)
    assert len(rep.pairs) == len(want) and (rep.pairs == want).all()
    assert rep.extra["batches"] >= (1 if mode == "filtered" else 11)
    assert rep.counters["candidates"] == 900 * 700 == rep.counters["verified"]
