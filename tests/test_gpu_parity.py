"""GPU parity: the B200 library through its C ABI versus the reference's own
outputs (tests/golden) and the C oracle.  Bit-exact: same sorted
(id_r, id_s, overlap) list, same counters, same saturated_records."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, golden_collection
from paper_1711_07295_b200 import capi, datasets as D
from paper_1711_07295_b200 import ssjoin as S

pytestmark = pytest.mark.gpu

COUNTER_KEYS = ("candidates", "pruned_length", "pruned_positional", "pruned_suffix", "pruned_bitmap",
                "bitmap_tested", "filter_evaluations", "verified", "matched")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def colls(lib, golden_arrays):
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = S.Collection.from_csr(lib, *golden_collection(golden_arrays, name))
        return cache[name]
    return get


def options_of(lib, e):
    o = S.default_options(lib)
    for k, v in e["options"].items():
        setattr(o, k, v)
    return o


def assert_same(rep, e, where=""):
    assert len(rep.pairs) == e["pair_count"], (where, e["label"])
    assert sha(rep.pairs) == e["pairs_sha256"], (where, e["label"])
    for k in COUNTER_KEYS:
        assert rep.counters[k] == e["counters"][k], (where, e["label"], k)
    assert rep.saturated_records == e["saturated_records"], (where, e["label"])


def test_sketch_kernel_matches_reference_stores(lib, golden, colls):
    for e in golden["bitmaps"]:
        store = S.build_bitmaps(colls(e["collection"]), e["method"], e["width"], e["hash"])
        assert sha(store) == e["sha256"], e


FILTERS = ["tc-fp4", "tc-i8-pair", "tc-i8", "tc-i8-1tile", "tc-i8-noext", "popc", "tc-l2gemm", "tc-head",
           "tc-head-i8"]


def set_filter(monkeypatch, flavour):
    """tcgen05 fp4 / int8 CTA-pair / int8 single-CTA with two row tiles per column
    tile (default) or one (with the popcount extension block, or K = b) /
    level-2 GEMM, or POPC; tc-head / tc-head-i8: the level-2 GEMM with the
    head-overlap kernel (K3a, mxf4 / int8 operands) forced over every record
    of >= 3 tokens with a 256 / 128-token head."""
    head = flavour.startswith("tc-head")
    monkeypatch.setenv("SSJB_FILTER", "popc" if flavour == "popc" else "tc")
    monkeypatch.setenv("SSJB_L2GEMM", "1" if flavour == "tc-l2gemm" or head else "0")
    monkeypatch.setenv("SSJB_HEAD", "2" if head else "0")
    monkeypatch.setenv("SSJB_HEAD_MIN_SIZE", "3")
    monkeypatch.setenv("SSJB_HEAD_KIND", "i8" if flavour == "tc-head-i8" else "fp4")
    monkeypatch.setenv("SSJB_HEAD_K", "128" if flavour == "tc-head-i8" else "256")
    # column-chunk-major work-item claim order (default only above 262144 rows)
    ordered = flavour in ("tc-i8", "tc-l2gemm", "tc-head", "tc-head-i8", "tc-fp4")
    monkeypatch.setenv("SSJB_ORDER_MIN_ROWS", "1" if ordered else "1000000000")
    monkeypatch.setenv("SSJB_TC_KIND", "i8" if flavour.startswith("tc-i8") else "fp4")
    monkeypatch.setenv("SSJB_TC2", "1" if flavour == "tc-i8-pair" else "0")
    monkeypatch.setenv("SSJB_NOEXT", "1" if flavour == "tc-i8-noext" else "0")
    monkeypatch.setenv("SSJB_TCM", "0" if flavour in ("tc-i8-1tile", "tc-i8-noext") else "1")


@pytest.mark.parametrize("flavour", FILTERS)
def test_every_golden_join(lib, golden, colls, flavour, monkeypatch):
    """Every reference fixture, through each filter kernel (tcgen05 fp4 and int8
    GEMMs, POPC, tcgen05 with the level-2 GEMM)."""
    set_filter(monkeypatch, flavour)
    for e in golden["joins"]:
        rep = S.join(colls(e["collection"]), options_of(lib, e))
        assert_same(rep, e, flavour)


@pytest.mark.parametrize("chunks", ["2", "5"])
def test_two_phase_streamed_ingest(lib, golden, colls, chunks, monkeypatch):
    """Dense joins stream in two phases: the first chunk's work items are
    filtered (and verified) while the rest of the collection is in flight;
    every fixture with the head kernel forced, first chunks of 1/2 and 1/5 of
    the tokens, and the saturated-row rescan on its side stream and inline."""
    set_filter(monkeypatch, "tc-head")
    monkeypatch.setenv("SSJB_STREAM", "1")
    monkeypatch.setenv("SSJB_STREAM_MIN_ROWS", "1")
    monkeypatch.setenv("SSJB_STREAM_CHUNKS_BATCH", chunks)
    monkeypatch.setenv("SSJB_RESCAN_SIDE", "1" if chunks == "2" else "0")
    for e in golden["joins"]:
        rep = S.join(colls(e["collection"]), options_of(lib, e))
        assert_same(rep, e, "two-phase " + chunks)


@pytest.mark.parametrize("mode", ["1", "2"])
@pytest.mark.parametrize("flavour", ["tc-i8", "tc-i8-pair", "tc-fp4", "tc-head"])
def test_streamed_ingest(lib, golden, colls, flavour, mode, monkeypatch):
    """Every fixture with the collection streamed to the device in 3 row chunks
    (decode + sketches + operands of a chunk overlap the next chunk's transfer;
    mode 2 also launches each chunk's filter work items as it lands)."""
    set_filter(monkeypatch, flavour)
    monkeypatch.setenv("SSJB_STREAM", mode)
    monkeypatch.setenv("SSJB_STREAM_MIN_ROWS", "1")
    monkeypatch.setenv("SSJB_STREAM_CHUNKS", "3")
    for e in golden["joins"]:
        rep = S.join(colls(e["collection"]), options_of(lib, e))
        assert_same(rep, e, "streamed " + flavour)


def test_row_shards_add_up(lib, golden, colls):
    for e in golden["joins"]:
        if e["options"]["algorithm"] != capi.SSJ_ALGO_PAR_BITMAP or e["collection"].startswith("acc1_"):
            continue
        coll = colls(e["collection"])
        opts = options_of(lib, e)
        for parts in (2, 3):
            b = S.partition_rows(coll, opts, parts)
            reps = [S.join_rows(coll, opts, int(b[k]), int(b[k + 1])) for k in range(parts)]
            pairs = np.sort(np.concatenate([r.pairs for r in reps]), order=["id_r", "id_s"])
            assert sha(pairs) == e["pairs_sha256"], e["label"]
            for k in COUNTER_KEYS:
                assert sum(r.counters[k] for r in reps) == e["counters"][k], (e["label"], k)
            assert sum(r.saturated_records for r in reps) == e["saturated_records"]


@pytest.fixture
def shards(lib):
    """ssjb_set_shards_per_device for one test, restored afterwards."""
    def set_(k):
        assert lib.ssjb_set_shards_per_device(k) == capi.SSJ_OK
    yield set_
    lib.ssjb_set_shards_per_device(0)


@pytest.mark.parametrize("count", [2, 4, 8])
def test_shard_count_changes_nothing(lib, golden, colls, shards, count):
    """Worker-count invariance through the drop-in path (reference
    tests/test_parallel.cpp:37-59, tests/acceptance.cpp:297-336): ssj_join
    split into 2/4/8 row shards -- the multi-GPU partition, per-shard engines
    on persistent device workers, and the shard merge of capi.cpp -- returns
    every fixture's bytes and counters unchanged."""
    shards(count)
    for e in golden["joins"]:
        if e["options"]["algorithm"] != capi.SSJ_ALGO_PAR_BITMAP:
            continue
        rep = S.join(colls(e["collection"]), options_of(lib, e))
        assert_same(rep, e, f"{count} shards")
        assert rep.extra["devices"] == count


@pytest.mark.parametrize("flavour", FILTERS)
def test_random_collections_vs_oracle(lib, oracle, flavour, monkeypatch):
    set_filter(monkeypatch, flavour)
    rng = np.random.default_rng(2024)
    for trial in range(40):
        n = int(rng.integers(50, 1500))
        universe = int(rng.integers(20, 3000))
        mean = float(rng.uniform(2, 40))
        dist = int(rng.integers(0, 2))
        coll = S.Collection.generate(lib, n, mean, universe, int(rng.integers(1 << 30)), dist)
        t, o = coll.csr()
        p, q = [(1, 2), (3, 5), (2, 3), (7, 10), (4, 5), (9, 10), (1, 1), (1, 3)][trial % 8]
        width = int(rng.choice([64, 128, 192, 256, 320, 512, 1024]))
        method = int(rng.integers(0, 3))
        hsh = int(rng.integers(0, 2))
        cap = int(rng.choice([1, 2, 7, 64, 2048]))
        enabled = bool(rng.integers(0, 5))
        cutoff = int(rng.choice([oracle.INT64_MAX, 0, 5, 12, 30]))
        mode = capi.SSJ_CUTOFF_OFF if cutoff == oracle.INT64_MAX else capi.SSJ_CUTOFF_EXPLICIT
        opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_PAR_BITMAP, threshold=(p, q),
                                 bitmap_enabled=int(enabled), bitmap_method=method, bitmap_bits=width,
                                 bitmap_hash=hsh, cutoff_mode=mode, cutoff_value=cutoff,
                                 buffer_capacity=cap)
        rep = S.join(coll, opts)
        want, cnt = oracle.par_bitmap_join(t, o, p, q, enabled, method, width, hsh, cutoff, cap)
        assert (rep.pairs == want).all() and len(rep.pairs) == len(want), trial
        assert rep.counters["candidates"] == cnt["candidates"], trial
        assert rep.counters["pruned_bitmap"] == cnt["pruned_bitmap"], trial
        assert rep.counters["bitmap_tested"] == cnt["bitmap_tested"], trial
        assert rep.counters["verified"] == cnt["verified"], trial
        assert rep.counters["matched"] == cnt["matched"], trial
        assert rep.saturated_records == cnt["saturated_records"], trial


def test_naive_vs_oracle(lib, oracle):
    rng = np.random.default_rng(7)
    for trial in range(6):
        coll = S.Collection.generate(lib, int(rng.integers(100, 900)), 6, 40, trial + 1)
        t, o = coll.csr()
        tau = [(1, 2), (7, 10), (1, 1)][trial % 3]
        rep = S.join(coll, S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE, threshold=tau))
        want, cnt = oracle.naive_join(t, o, *tau)
        assert (rep.pairs == want).all() and len(rep.pairs) == len(want)
        assert rep.counters["candidates"] == cnt["candidates"] == rep.counters["verified"]


@pytest.mark.parametrize("flavour", ["default", "tc-head"])
def test_survivor_and_result_overflow_batches(lib, golden, colls, monkeypatch, flavour):
    """Tiny survivor/result buffers force many filter batches and result runs
    (tc-head: level-2 GEMM batches in column-chunk-major claim order, then
    head-overlap batches)."""
    if flavour != "default":
        set_filter(monkeypatch, flavour)
    monkeypatch.setenv("SSJB_SURVIVOR_CAP", str(1 << 19))
    monkeypatch.setenv("SSJB_RESULT_CAP", str(1 << 19))
    for e in golden["joins"]:
        if e["collection"] in ("dups_2500", "acc8_2000", "par_500") and e["pair_count"] > 0:
            rep = S.join(colls(e["collection"]), options_of(lib, e))
            assert_same(rep, e, "overflow")
    e = next(x for x in golden["joins"] if x["collection"] == "dups_2500")
    rep = S.join(colls("dups_2500"), options_of(lib, e))
    assert rep.extra["batches"] > 1


def test_pinned_replica_and_repeat_determinism(lib, golden, colls):
    e = next(x for x in golden["joins"] if x["label"] == "acceptance criterion 8")
    coll = colls(e["collection"])
    S.pin_device(coll, 0)
    try:
        for _ in range(3):
            assert_same(S.join(coll, options_of(lib, e)), e, "pinned")
    finally:
        S.unpin_device(coll, 0)
    assert_same(S.join(coll, options_of(lib, e)), e, "unpinned")


def _large():
    path = os.path.join(GOLDEN_DIR, "large.jsonl")
    if not os.path.exists(path):
        return []
    # C1/C2 here; the heavy-tailed configs (C3...) are checked in test_gpu_heavy.py
    return [e for e in map(json.loads, open(path)) if e["case"] == "C1" or e["case"].startswith("C2_")]


@pytest.mark.parametrize("case", [c["case"] for c in _large()] or ["none"])
def test_full_size_configs_match_reference(lib, case):
    """BASELINE configs at full size vs the reference library's own run."""
    entries = {c["case"]: c for c in _large()}
    if case not in entries:
        pytest.skip("no full-size fixtures")
    e = entries[case]
    coll = D.c1(lib) if case == "C1" else _c2(lib)
    opts = S.par_bitmap_options(lib, threshold=tuple(e["tau"]), method=capi.SSJ_BITMAP_XOR,
                                bits=e["bits"], cutoff_mode=capi.SSJ_CUTOFF_OFF)
    rep = S.join(coll, opts)
    assert len(rep.pairs) == e["pair_count"]
    assert sha(rep.pairs) == e["pairs_sha256"]
    for k in COUNTER_KEYS:
        assert rep.counters[k] == e["counters"][k], k
    assert rep.saturated_records == e["saturated_records"]


_C2 = {}


def _c2(lib):
    if "c" not in _C2:
        _C2["c"] = D.c2(lib)
    return _C2["c"]


@pytest.mark.parametrize("flavour", ["tc-l2gemm", "tc-i8"])
def test_level3_verify_filter(lib, golden, colls, flavour, monkeypatch):
    """Every fixture with the level-3 (512-bit Xor) re-test applied to every
    survivor before the merge (dense joins enable it in their batch phase):
    it may only drop pairs that cannot match."""
    set_filter(monkeypatch, flavour)
    monkeypatch.setenv("SSJB_L3_FORCE", "1")
    monkeypatch.setenv("SSJB_L3_MIN", "0")
    for e in golden["joins"]:
        rep = S.join(colls(e["collection"]), options_of(lib, e))
        assert_same(rep, e, flavour + "+l3")


def test_concurrent_joins_from_threads(lib, golden, colls):
    """Joins from four host threads at once (each on its own stream, sharing
    collections, pinned replicas and the workspace pool) give every fixture's
    exact result -- bench.py runs the sweep's joins two at a time."""
    from concurrent.futures import ThreadPoolExecutor
    cases = [e for e in golden["joins"] if e["options"]["algorithm"] == 6][:120]
    work = [(colls(e["collection"]), options_of(lib, e)) for e in cases]  # (npz reads stay on this thread)
    pinned = work[0][0]
    S.pin_device(pinned)
    try:
        with ThreadPoolExecutor(max_workers=4) as pool:
            reps = list(pool.map(lambda w: S.join(w[0], w[1]), work))
    finally:
        S.unpin_device(pinned)
    for rep, e in zip(reps, cases):
        assert_same(rep, e, "concurrent")


@pytest.mark.parametrize("sim", [capi.SSJ_SIM_JACCARD, capi.SSJ_SIM_COSINE, capi.SSJ_SIM_DICE,
                                 capi.SSJ_SIM_OVERLAP])
def test_prefix_filter_algorithm_codes_return_the_reference_pairs(lib, ref, sim):
    """ssj_join with ALLPAIRS / PPJOIN / PPJOIN+ / GROUPJOIN / ADAPTJOIN (the
    GPU prefix-filter engine) returns the reference's pair list AND all nine
    counters for that algorithm (run live from oracle/_ref on the same
    collection and options) for every similarity function, bitmap off / on
    (filter3) / filter2."""
    rng = np.random.default_rng(77 + sim)
    for trial in range(6):
        n = int(rng.integers(100, 900))
        gen = dict(num_sets=n, mean_size=float(rng.uniform(4, 30)), universe=int(rng.integers(30, 400)),
                   seed=int(rng.integers(0, 1 << 30)))
        mine = S.Collection.generate(lib, **gen)
        theirs = S.Collection.generate(ref, **gen)
        thr = (int(rng.integers(2, 8)), 1) if sim == capi.SSJ_SIM_OVERLAP else (int(rng.integers(4, 10)), 10)
        for algo in (1, 2, 3, 4, 5):
            kw = dict(algorithm=algo, similarity=sim, threshold=thr, bitmap_enabled=int(trial % 3 != 0),
                      placement=capi.SSJ_PLACEMENT_FILTER2 if trial % 3 == 2 else capi.SSJ_PLACEMENT_DEFAULT,
                      workers=2)
            want = S.join(theirs, S.default_options(ref, **kw))
            got = S.join(mine, S.default_options(lib, **kw))
            assert len(got.pairs) == len(want.pairs) and (got.pairs == want.pairs).all(), (sim, algo, trial)
            c = got.counters
            assert c["candidates"] == (c["pruned_length"] + c["pruned_positional"] + c["pruned_suffix"]
                                       + c["pruned_bitmap"] + c["verified"])
            assert c["matched"] == len(got.pairs)
            assert c == want.counters, (sim, algo, trial)


@pytest.mark.parametrize("tiers", ["1", "0"])
@pytest.mark.parametrize("mean", [3.0, 40.0, 400.0])
def test_sketch_build_heavy_tail(lib, oracle, mean, tiers, monkeypatch):
    """Heavy-tailed sizes: the build runs in size tiers (2^k lanes per record,
    a warp, one CTA per record for the tail rows: build_sketches_big), or as
    one launch (SSJB_BUILD_ONE_TIER=1); every Set / Xor store (with and without
    the multiplicative hash, 64..512 bits) equals the oracle's
    (reference src/bitmap.cpp:66-88,145-158)."""
    monkeypatch.setenv("SSJB_BUILD_ONE_TIER", "0" if tiers == "1" else "1")
    rng = np.random.default_rng(int(mean))
    n = 3000
    sizes = np.minimum(np.maximum(1, rng.lognormal(np.log(mean), 1.2, n).astype(np.int64)), 20000)
    sizes[-5:] = [5000, 9000, 12000, 17000, 20000]
    recs = [np.unique(rng.integers(0, 200000, int(z))).tolist() for z in sizes]
    coll = S.Collection.from_records(lib, recs)
    t, o = coll.csr()
    for method in (capi.SSJ_BITMAP_SET, capi.SSJ_BITMAP_XOR):
        for bits, h in ((64, 0), (128, 1), (256, 0), (512, 1)):
            got = S.build_bitmaps(coll, method, bits, h)
            want = oracle.build_bitmaps(t, o, method, bits, h)
            assert (got == want).all(), (mean, method, bits, h)
