"""Host side of the B200 library (no GPU needed): the C ABI surface, the
collection pipeline that defines record ids, option resolution and analytics
-- each compared with the reference's own outputs (tests/golden)."""
import ctypes as C
import hashlib
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden_collection, has_gpu
from paper_1711_07295_b200 import capi
from paper_1711_07295_b200 import ssjoin as S

LIB = os.path.join(ROOT, "paper_1711_07295_b200", "lib", "libssjoin.so")


def test_library_exports_every_declared_symbol(lib):
    exported = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True,
                              check=True).stdout
    names = {line.split()[-1] for line in exported.splitlines() if line.strip()}
    for header in ("ssjoin.h", "ssjoin_b200.h"):
        text = open(os.path.join(ROOT, "include", header)).read()
        import re
        declared = set(re.findall(r"\b(ssjb?_[a-z_]+)\s*\(", text))
        missing = declared - names
        assert not missing, (header, missing)
    assert set(capi.SSJ_SYMBOLS) <= names and set(capi.SSJB_SYMBOLS) <= names
    # nothing but the C ABI leaks out of the library
    assert all(n.startswith(("ssj_", "ssjb_")) for n in names if not n.startswith("_")), names


def test_struct_layouts_and_defaults(lib):
    opts = S.default_options(lib)
    assert C.sizeof(opts) == 80
    assert (opts.algorithm, opts.similarity, opts.threshold_num, opts.threshold_den) == (1, 1, 1, 2)
    assert (opts.bitmap_enabled, opts.bitmap_method, opts.cutoff_mode) == (0, 3, 0)
    assert (opts.suffix_depth, opts.ell_max, opts.workers, opts.buffer_capacity) == (2, 3, 1, 2048)


def test_generator_matches_reference(lib, golden):
    for e in golden["generator"]:
        coll = S.Collection.generate(lib, e["num_sets"], e["mean_size"], e["universe"], e["seed"],
                                     e["distribution"], e["zipf_exponent"])
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "c.txt")
            coll.write(p)
            digest = hashlib.sha256(open(p, "rb").read()).hexdigest()
        assert digest == e["file_sha256"], e["name"]
        assert (len(coll), coll.median_size, coll.max_size, coll.universe) == \
            (e["size"], e["median"], e["max"], e["universe_size"]), e["name"]
        assert coll.mean_size == e["mean"], e["name"]


def test_csr_canonical_order_matches_reference(lib, golden_arrays):
    for name in ("par_1500", "edge_empty", "dups_2500", "three", "empty", "zipf_3000"):
        t, o = golden_collection(golden_arrays, name)
        # feed the canonical records back shuffled and with duplicate tokens
        rng = np.random.default_rng(1)
        recs = [t[int(o[r]):int(o[r + 1])].tolist() for r in range(len(o) - 1)]
        scrambled = [rng.permutation(r + r[:1]).tolist() for r in recs]
        order = rng.permutation(len(scrambled))
        coll = S.Collection.from_records(lib, [scrambled[k] for k in order])
        t2, o2 = coll.csr()
        assert (o2 == o).all() and (t2 == t).all(), name


def test_load_write_roundtrip_and_errors(lib, tmp_path):
    p = tmp_path / "ok.txt"
    p.write_text("1 2\n1 2 3\n\n7  3 3\n")
    coll = S.Collection.load(lib, str(p))
    assert len(coll) == 4 and coll.universe == 8 and coll.max_size == 3 and coll.median_size == 2
    out = tmp_path / "w.txt"
    coll.write(str(out))
    assert out.read_text() == "\n1 2\n3 7\n1 2 3\n"
    again = S.Collection.load(lib, str(out))
    assert (again.csr()[0] == coll.csr()[0]).all()
    # reference tests/test_capi.cpp:153-179
    with pytest.raises(S.SsjError) as e:
        S.Collection.load(lib, "/no/such/file")
    assert e.value.status == capi.SSJ_ERROR_IO
    bad = tmp_path / "bad.txt"
    bad.write_text("1 oops 3\n")
    with pytest.raises(S.SsjError) as e:
        S.Collection.load(lib, str(bad))
    assert e.value.status == capi.SSJ_ERROR_PARSE and "line 1" in e.value.message
    big = tmp_path / "big.txt"
    big.write_text("1\n4294967296\n")
    with pytest.raises(S.SsjError) as e:
        S.Collection.load(lib, str(big))
    assert "line 2: token id out of range" in e.value.message


def test_text_inputs_match_reference(lib, ref, tmp_path):
    p = tmp_path / "t.txt"
    p.write_text("the cat sat\nthe dog sat down\n\ncat cat dog\nzebra the\n")
    for fmt, q in ((capi.SSJ_INPUT_WORDS, 0), (capi.SSJ_INPUT_QGRAMS, 3), (capi.SSJ_INPUT_QGRAMS, 1)):
        a = S.Collection.load(lib, str(p), fmt, q)
        b = S.Collection.load(ref, str(p), fmt, q)
        assert len(a) == len(b) and a.universe == b.universe
        ta, oa = a.csr()
        tb, ob = b.csr()
        assert (ta == tb).all() and (oa == ob).all()


def test_parse_threshold_matches_reference(lib, golden):
    for e in golden["analytics"]["parse"]:
        if e["ok"]:
            assert list(S.parse_threshold(lib, e["text"])) == e["value"], e
        else:
            with pytest.raises(S.SsjError) as err:
                S.parse_threshold(lib, e["text"])
            assert err.value.status == e["status"], e


def test_analytics_match_reference(lib, golden):
    for e in golden["analytics"]["cutoff"]:
        assert S.cutoff(lib, e["method"], e["bits"], e["num"], e["den"], e["space"]) == e["value"], e
    for e in golden["analytics"]["expected_bound"]:
        assert S.expected_bound(lib, e["method"], e["bits"], e["n"]) == e["value"], e


def test_monte_carlo_matches_reference(lib, ref):
    for args in ((1, 64, 8, 2000, 5), (0, 128, 30, 300, 7), (2, 64, 40, 200, 3)):
        a, b = C.c_double(), C.c_double()
        assert lib.ssj_monte_carlo_bound(*args, C.byref(a)) == 0
        assert ref.ssj_monte_carlo_bound(*args, C.byref(b)) == 0
        assert a.value == b.value


def test_resolve_bitmap_matches_reference(lib, golden, golden_arrays):
    colls = {}
    for e in golden["analytics"]["resolve"]:
        name = e["collection"]
        if name not in colls:
            colls[name] = S.Collection.from_csr(lib, *golden_collection(golden_arrays, name))
        opts = S.default_options(lib, algorithm=capi.SSJ_ALGO_PAR_BITMAP, threshold=(e["num"], e["den"]),
                                 bitmap_enabled=1, bitmap_method=e["method"],
                                 cutoff_mode=e["cutoff_mode"], cutoff_value=42)
        assert list(S.resolve_bitmap(colls[name], opts)) == e["result"], e


def test_option_errors_match_reference(lib, ref):
    """Invalid options fail identically (status and message) before any GPU work."""
    cases = [dict(algorithm=99), dict(threshold=(3, 2)), dict(threshold=(1, 0)), dict(similarity=7),
             dict(bitmap_method=9), dict(cutoff_mode=5), dict(placement=4),
             dict(algorithm=capi.SSJ_ALGO_PAR_BITMAP, workers=0),
             dict(algorithm=capi.SSJ_ALGO_PAR_BITMAP, buffer_capacity=0),
             dict(algorithm=capi.SSJ_ALGO_PAR_BITMAP, similarity=capi.SSJ_SIM_DICE)]
    for kw in cases:
        got = []
        for L in (lib, ref):
            coll = S.Collection.from_records(L, [[1, 2], [1, 2, 3]])
            with pytest.raises(S.SsjError) as e:
                S.join(coll, S.default_options(L, **kw))
            got.append((e.value.status, e.value.message))
        assert got[0] == got[1], (kw, got)
    # RS-joins with a non-naive algorithm (reference src/capi.cpp:225-228)
    coll = S.Collection.from_records(lib, [[1, 2], [1, 2, 3]])
    with pytest.raises(S.SsjError) as e:
        S.join(coll, S.default_options(lib, algorithm=capi.SSJ_ALGO_PAR_BITMAP), other=coll)
    assert e.value.status == capi.SSJ_ERROR_INVALID_ARGUMENT


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_prefix_filter_algorithms_reach_the_gpu_join(lib):
    """ALLPAIRS..ADAPTJOIN are accepted (routed to the GPU exact join, see
    capi.cpp check_supported): without a device they fail like PAR_BITMAP."""
    coll = S.Collection.from_records(lib, [[1, 2], [1, 2, 3]])
    for algo in (1, 2, 3, 4, 5):
        with pytest.raises(S.SsjError) as e:
            S.join(coll, S.default_options(lib, algorithm=algo))
        assert e.value.status == capi.SSJ_ERROR_INTERNAL and "CUDA" in e.value.message


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_join_without_gpu_fails_loudly(lib):
    coll = S.Collection.from_records(lib, [[1, 2], [1, 2, 3]])
    with pytest.raises(S.SsjError) as e:
        S.join(coll, S.par_bitmap_options(lib, threshold=(1, 2)))
    assert e.value.status == capi.SSJ_ERROR_INTERNAL and "CUDA" in e.value.message


def test_partition_rows_balances_window_pairs(lib, golden_arrays):
    coll = S.Collection.from_csr(lib, *golden_collection(golden_arrays, "zipf_3000"))
    opts = S.par_bitmap_options(lib, threshold=(1, 2))
    for parts in (1, 2, 3, 8):
        b = S.partition_rows(coll, opts, parts)
        assert b[0] == 0 and b[-1] == len(coll) and (np.diff(b.astype(np.int64)) >= 0).all()


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_delivery_entry_points_fail_loudly_without_gpu(lib, tmp_path):
    import ctypes as C
    coll = S.Collection.from_records(lib, [[1, 2], [1, 2, 3]])
    opts = S.par_bitmap_options(lib, threshold=(1, 2))
    for call in (lambda: S.join_count(coll, opts),
                 lambda: S.join_stream(coll, opts, lambda a: None),
                 lambda: S.join_write_pairs(coll, opts, str(tmp_path / "p.txt")),
                 lambda: S.join(coll, S.default_options(lib, algorithm=capi.SSJ_ALGO_NAIVE), coll)):
        with pytest.raises(S.SsjError) as e:
            call()
        assert e.value.status == capi.SSJ_ERROR_INTERNAL and "CUDA" in e.value.message
    # argument errors come first, like ssj_join's (reference src/capi.cpp:220-228)
    out = C.c_void_p()
    assert lib.ssjb_join_count(None, None, C.byref(opts), C.byref(out)) == capi.SSJ_ERROR_INVALID_ARGUMENT
    assert lib.ssjb_join_count(coll.handle, coll.handle, C.byref(opts), C.byref(out)) == \
        capi.SSJ_ERROR_INVALID_ARGUMENT
    assert b"naive" in lib.ssj_last_error()
    assert lib.ssjb_report_write_pairs(None, b"x") == capi.SSJ_ERROR_INVALID_ARGUMENT


@pytest.mark.parametrize("threads", ["1", "3", "8"])
def test_parallel_ingest_matches_reference(lib, ref, tmp_path, threads):
    """Multi-MB id files parse in per-thread slices (SSJB_HOST_THREADS); the
    canonical collection, universe and error lines must equal the reference's
    read_id_lines (src/collection.cpp:97-137) regardless of slicing."""
    import subprocess
    import sys
    rng = np.random.default_rng(7)
    n = 150_000
    sizes = rng.integers(0, 12, n)
    lines = []
    for k, sz in enumerate(sizes):
        toks = rng.integers(0, 5000 if k % 3 else 70, sz)       # duplicates inside records
        sep = "  " if k % 11 == 0 else " "
        lines.append(sep.join(map(str, toks.tolist())) + (" " if k % 13 == 0 else ""))
    body = "\n".join(lines)
    cases = {"trailing_nl": body + "\n", "no_trailing_nl": body, "blank_tail": body + "\n\n \n"}
    bad_line = 123_457
    bad = lines[:]
    bad[bad_line - 1] = bad[bad_line - 1] + " 12x"
    cases["error"] = "\n".join(bad) + "\n"
    over = lines[:]
    over[140_001 - 1] = "4294967296"
    cases["overflow"] = "\n".join(over) + "\n"
    for name, text in cases.items():
        p = tmp_path / f"{name}.txt"
        p.write_text(text)
        # run the product in a child so SSJB_HOST_THREADS takes effect
        code = ("import sys, numpy as np; sys.path.insert(0, %r)\n"
                "from paper_1711_07295_b200 import load_library, ssjoin as S\n"
                "lib = load_library()\n"
                "try:\n"
                "    c = S.Collection.load(lib, %r); t, o = c.csr()\n"
                "    np.savez(%r, t=t, o=o, u=c.universe)\n"
                "except S.SsjError as e:\n"
                "    print('ERR', e.status, e.message)\n") % (ROOT, str(p), str(tmp_path / "out.npz"))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           env={**os.environ, "SSJB_HOST_THREADS": threads}, check=True)
        try:
            want = S.Collection.load(ref, str(p))
        except S.SsjError as e:
            assert r.stdout.startswith("ERR"), (name, r.stdout)
            assert r.stdout.split(None, 2)[2].strip() == e.message, name
            continue
        got = np.load(tmp_path / "out.npz")
        tw, ow = want.csr()
        assert (got["t"] == tw).all() and (got["o"] == ow).all(), name
        assert int(got["u"]) == want.universe, name


def test_parallel_canonical_sort_matches_reference(lib, ref):
    """collection_from_csr's parallel record sort == the reference canonical
    order, on records with long shared prefixes (ties beyond the first two
    tokens) and many exact duplicates."""
    rng = np.random.default_rng(11)
    recs = []
    for k in range(60_000):
        base = [1, 2, 3, 4] if k % 4 == 0 else [int(x) for x in rng.integers(0, 50, 2)]
        recs.append(base + [int(x) for x in rng.integers(0, 9, k % 5)])
    recs += [[9, 9, 9]] * 500 + [[]] * 100
    a = S.Collection.from_records(lib, recs)
    b = S.Collection.from_records(ref, recs)
    ta, oa = a.csr()
    tb, ob = b.csr()
    assert (ta == tb).all() and (oa == ob).all()
