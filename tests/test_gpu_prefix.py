"""GPU prefix-filter joins against the reference's own runs.

ssj_join with ALLPAIRS / PPJOIN / PPJOIN+ / GROUPJOIN / ADAPTJOIN runs the
GPU prefix-filter engine (csrc/prefix_join.cuh): every case of
tests/golden/golden_prefix.json (made by make_golden_prefix.py from the
unmodified reference, src/join.cpp:132-420) must give the same sorted pair
list and the same nine counters -- the algorithm-specific ones included
(filter_evaluations, pruned_length / positional / suffix, bitmap_tested)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from paper_1711_07295_b200 import capi
from paper_1711_07295_b200 import ssjoin as S


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gp():
    with open(os.path.join(GOLDEN_DIR, "golden_prefix.json")) as f:
        cases = json.load(f)["cases"]
    return cases, np.load(os.path.join(GOLDEN_DIR, "golden_prefix.npz"))


def options_of(lib, case):
    o = S.default_options(lib)
    for k, v in case["options"].items():
        setattr(o, k, v)
    return o


def test_prefix_fixtures_are_consistent(gp):
    """CPU: the committed fixtures hold the reference's counter invariants
    (tests/test_joins.cpp:14-19) and their stored pair arrays match the shas."""
    cases, arr = gp
    algos = set()
    for c in cases:
        k = c["counters"]
        assert k["candidates"] == (k["pruned_length"] + k["pruned_positional"] + k["pruned_suffix"] +
                                   k["pruned_bitmap"] + k["verified"]), c["id"]
        assert k["matched"] == c["pair_count"]
        if f"pairs/{c['id']}" in arr:
            assert sha(arr[f"pairs/{c['id']}"]) == c["pairs_sha256"]
        algos.add(c["options"]["algorithm"])
    assert algos == {1, 2, 3, 4, 5}
    assert any(c["counters"]["pruned_suffix"] for c in cases)
    assert any(c["counters"]["pruned_positional"] for c in cases)
    assert any(c["counters"]["pruned_bitmap"] and c["options"]["placement"] == 1 for c in cases)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", [1, 2, 3, 4, 5])
def test_prefix_joins_match_reference_fixtures(lib, gp, algo):
    cases, arr = gp
    colls = {}
    n = 0
    for c in cases:
        if c["options"]["algorithm"] != algo:
            continue
        name = c["collection"]
        if name not in colls:
            colls[name] = S.Collection.from_csr(lib, arr[f"coll/{name}/tokens"], arr[f"coll/{name}/offsets"])
        rep = S.join(colls[name], options_of(lib, c))
        where = (c["id"], c["label"], c["collection"])
        assert rep.counters == c["counters"], (where, rep.counters, c["counters"])
        assert len(rep.pairs) == c["pair_count"], where
        assert sha(rep.pairs) == c["pairs_sha256"], where
        n += 1
    assert n > 200


@pytest.mark.gpu
def test_prefix_joins_survive_result_overflow(lib, gp, monkeypatch):
    """A result buffer smaller than the output (SSJB_PREFIX_RESULT_CAP) makes
    the engine re-run with the exact size, and an AdaptJoin candidate list that
    does not fit (SSJB_ADAPT_LIST_CAP) falls back to re-enumerating the
    encounters: same pairs and counters."""
    cases, arr = gp
    monkeypatch.setenv("SSJB_PREFIX_RESULT_CAP", "1000")
    monkeypatch.setenv("SSJB_ADAPT_LIST_CAP", "3")  # AdaptJoin: verify by re-enumeration
    done = set()
    for c in cases:
        algo = c["options"]["algorithm"]
        if algo in done or not 5000 < c["pair_count"] < 200000:
            continue
        name = c["collection"]
        coll = S.Collection.from_csr(lib, arr[f"coll/{name}/tokens"], arr[f"coll/{name}/offsets"])
        rep = S.join(coll, options_of(lib, c))
        assert rep.counters == c["counters"], c["id"]
        assert sha(rep.pairs) == c["pairs_sha256"], c["id"]
        done.add(algo)
    assert done == {1, 2, 3, 4, 5}


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_prefix_joins_full_size(lib, name):
    """Full-size BASELINE-shaped collections (C1 tau 0.9, C2 tau 0.8, C3 tau
    0.5 with 203.6M pairs, C4 tau 0.7 with 42.4M pairs): pairs sha256 and all
    nine counters equal the reference's own single-threaded runs
    (tests/golden/prefix_large.jsonl, make_golden_prefix_large.py)."""
    from paper_1711_07295_b200 import datasets as D
    with open(os.path.join(GOLDEN_DIR, "prefix_large.jsonl")) as f:
        cases = [json.loads(l) for l in f if l.strip()]
    cases = [c for c in cases if c["config"] == name]
    assert cases
    coll = getattr(D, name)(lib)
    t, o = coll.csr()
    assert hashlib.sha256(np.ascontiguousarray(t).tobytes() + np.ascontiguousarray(o).tobytes()).hexdigest() == \
        cases[0]["collection_sha256"]
    for c in cases:
        rep = S.join(coll, options_of(lib, c))
        where = (name, c["algo"], c["bitmap"])
        assert rep.counters == c["counters"], (where, rep.counters, c["counters"])
        assert len(rep.pairs) == c["pair_count"] and sha(rep.pairs) == c["pairs_sha256"], where
        del rep


@pytest.mark.gpu
def test_prefix_joins_delivery_entry_points(lib, gp):
    """ssjb_join_count and ssjb_join_stream take the prefix-filter codes too:
    the same counters, and the streamed chunks concatenate to the pair list."""
    cases, arr = gp
    seen = set()
    for c in cases:
        algo = c["options"]["algorithm"]
        if algo in seen or c["pair_count"] < 50:
            continue
        seen.add(algo)
        name = c["collection"]
        coll = S.Collection.from_csr(lib, arr[f"coll/{name}/tokens"], arr[f"coll/{name}/offsets"])
        o = options_of(lib, c)
        assert S.join_count(coll, o).counters == c["counters"], c["id"]
        chunks = []
        rep = S.join_stream(coll, o, lambda a: chunks.append(a.copy()), chunk_pairs=17)
        assert rep.counters == c["counters"], c["id"]
        got = np.concatenate(chunks) if chunks else np.zeros(0, dtype=S.PAIR_DTYPE)
        assert len(got) == c["pair_count"] and sha(got) == c["pairs_sha256"], c["id"]
    assert seen == {1, 2, 3, 4, 5}
