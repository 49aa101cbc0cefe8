"""Result delivery beyond ssj_join's materialised list:
streaming chunks in canonical order (ssjb_join_stream), count-first
(ssjb_join_count) and the reference CLI's text pairs format
(ssjb_join_write_pairs / ssjb_report_write_pairs, reference
tools/ssjoin_cli.cpp:290-294).  Every variant must reproduce ssj_join's pairs
and counters exactly -- ssj_join itself is pinned to the reference by
test_gpu_parity.py."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1711_07295_b200 import capi
from paper_1711_07295_b200 import ssjoin as S

pytestmark = pytest.mark.gpu

COUNTERS = ("candidates", "pruned_bitmap", "bitmap_tested", "verified", "matched")


def text_of(pairs):
    return "".join(f"{int(p['id_r'])} {int(p['id_s'])} {int(p['overlap'])}\n" for p in pairs)


@pytest.fixture(scope="module")
def dense(lib):
    # small universe: ~1e5+ result pairs at tau 1/2
    return S.Collection.generate(lib, 3000, 10, 25, 5)


def _stream(coll, opts, other=None, chunk_pairs=0):
    chunks = []
    rep = S.join_stream(coll, opts, lambda a: chunks.append(a.copy()), other, chunk_pairs)
    return rep, chunks


@pytest.fixture(scope="module")
def denser(lib):
    return S.Collection.generate(lib, 8000, 10, 25, 6)


@pytest.mark.parametrize("env", [{}, {"SSJB_SURVIVOR_CAP": "1", "SSJB_RESULT_CAP": "1"}])
@pytest.mark.parametrize("chunk_pairs", [0, 7000, 1])
def test_stream_equals_join(lib, dense, denser, monkeypatch, env, chunk_pairs):
    """With the minimum (1M) survivor and result buffers and the bitmap off,
    every window pair is a survivor: the join runs in many batches and leaves
    several sorted runs in HBM; the per-chunk GPU merge must still produce
    ssj_join's list in order."""
    coll = denser if env else dense
    opts = (S.default_options(lib, algorithm=capi.SSJ_ALGO_PAR_BITMAP, threshold=(1, 2)) if env
            else S.par_bitmap_options(lib, threshold=(1, 2), bits=64))
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    want = S.join(coll, opts)
    assert len(want.pairs) > 50000
    rep, chunks = _stream(coll, opts, chunk_pairs=chunk_pairs)
    got = np.concatenate(chunks)
    assert got.tobytes() == want.pairs.tobytes()
    if chunk_pairs:
        # chunks hold whole id_r ranges of about chunk_pairs pairs
        assert len(chunks) > 1
        for a, b in zip(chunks, chunks[1:]):
            assert a["id_r"][-1] < b["id_r"][0]
        big = [c for c in chunks if len(c) > chunk_pairs]
        assert all((c["id_r"] == c["id_r"][0]).all() for c in big)
    for k in COUNTERS:
        assert rep.counters[k] == want.counters[k], k
    assert rep.saturated_records == want.saturated_records
    assert len(rep.pairs) == 0
    if env:
        assert rep.extra["batches"] > 10 and rep.counters["verified"] > 10 * (1 << 20)


def test_count_first(lib, dense, monkeypatch):
    for opts in (S.par_bitmap_options(lib, threshold=(1, 2), bits=64),
                 S.par_bitmap_options(lib, threshold=(7, 10), bits=128),
                 S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE, threshold=(3, 5))):
        want = S.join(dense, opts)
        rep = S.join_count(dense, opts)
        assert len(rep.pairs) == 0
        assert rep.counters == want.counters
        assert rep.saturated_records == want.saturated_records
        assert rep.counters["matched"] == len(want.pairs)
    monkeypatch.setenv("SSJB_SURVIVOR_CAP", "1")
    monkeypatch.setenv("SSJB_RESULT_CAP", "1")
    opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_PAR_BITMAP, threshold=(1, 2))
    assert S.join_count(dense, opts).counters == S.join(dense, opts).counters


def test_rs_stream_and_count(lib, monkeypatch):
    r = S.Collection.generate(lib, 1200, 8, 20, 41)
    s = S.Collection.generate(lib, 900, 8, 20, 42)
    opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE, threshold=(1, 2))
    want = S.join(r, opts, s)
    assert len(want.pairs) > 10000
    monkeypatch.setenv("SSJB_RS_BATCH", "100000")
    rep, chunks = _stream(r, opts, s, chunk_pairs=3000)
    assert np.concatenate(chunks).tobytes() == want.pairs.tobytes()
    assert rep.counters == want.counters
    assert S.join_count(r, opts, s).counters == want.counters


def test_write_pairs_text_format(lib, dense, tmp_path, monkeypatch):
    opts = S.par_bitmap_options(lib, threshold=(3, 5), bits=64)
    want = S.join(dense, opts)
    path = str(tmp_path / "pairs.txt")
    rep = S.join_write_pairs(dense, opts, path)
    assert open(path).read() == text_of(want.pairs)
    assert rep.counters == want.counters
    # materialised report -> same text (ssjb_report_write_pairs)
    out = C.c_void_p()
    assert lib.ssj_join(dense.handle, None, C.byref(opts), C.byref(out)) == capi.SSJ_OK
    p2 = str(tmp_path / "pairs2.txt")
    assert lib.ssjb_report_write_pairs(out, os.fsencode(p2)) == capi.SSJ_OK
    lib.ssj_report_free(out)
    assert open(p2).read() == open(path).read()
    # unwritable path -> SSJ_ERROR_IO
    with pytest.raises(S.SsjError) as ei:
        S.join_write_pairs(dense, opts, str(tmp_path / "no_such_dir" / "x.txt"))
    assert ei.value.status == capi.SSJ_ERROR_IO


def test_sink_can_stop_the_join(lib, dense):
    opts = S.par_bitmap_options(lib, threshold=(1, 2), bits=64)
    seen = []

    def stop(a):
        seen.append(len(a))
        return True
    with pytest.raises(S.SsjError) as ei:
        S.join_stream(dense, opts, stop, chunk_pairs=1000)
    assert ei.value.status == capi.SSJ_ERROR_IO
    assert len(seen) == 1


def test_golden_pairs_text(lib, golden, golden_arrays, tmp_path):
    """Text output of reference fixtures equals the CLI formatting of the
    reference's own pairs."""
    from conftest import golden_collection
    done = 0
    for e in golden["joins"]:
        key = f"pairs/{e['id']}"
        if e["pair_count"] < 5 or key not in golden_arrays.files or e["options"]["algorithm"] != 6:
            continue
        coll = S.Collection.from_csr(lib, *golden_collection(golden_arrays, e["collection"]))
        opts = S.default_options(lib)
        for k, v in e["options"].items():
            setattr(opts, k, v)
        path = str(tmp_path / f"{e['id']}.txt")
        S.join_write_pairs(coll, opts, path)
        assert open(path).read() == text_of(golden_arrays[key]), e["label"]
        done += 1
        if done >= 12:
            break
    assert done >= 5


def test_delivery_with_empty_outputs(lib, tmp_path):
    """No pairs at all (and an empty collection): no chunk is delivered, the
    text file is empty, counters still match ssj_join's."""
    for recs in ([[1, 2, 3], [4, 5, 6], [7, 8, 9, 10]], [], [[]] * 4):
        coll = S.Collection.from_records(lib, recs)
        opts = S.par_bitmap_options(lib, threshold=(9, 10), bits=64)
        want = S.join(coll, opts)
        assert len(want.pairs) == 0
        rep, chunks = _stream(coll, opts, chunk_pairs=10)
        assert chunks == [] and rep.counters == want.counters
        assert S.join_count(coll, opts).counters == want.counters
        path = str(tmp_path / "empty.txt")
        S.join_write_pairs(coll, opts, path)
        assert open(path).read() == ""
