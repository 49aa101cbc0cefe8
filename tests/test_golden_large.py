"""Consistency of the full-size reference fixtures (tests/golden/large.jsonl).

C4 and C5 are too large for the reference's PAR_BITMAP on a CPU, so their
full pair lists come from the reference's exact PPJOIN
(tests/golden/make_golden_exact.py); every exact algorithm returns the
PAR_BITMAP pair list (reference proj/tests/test_joins.cpp:62-112).  This test
pins that method on C3, where both reference runs exist: the PPJOIN pair
list must be byte-identical to the PAR_BITMAP one."""
import json
import os

from conftest import GOLDEN_DIR


def load():
    out = {}
    for line in open(os.path.join(GOLDEN_DIR, "large.jsonl")):
        e = json.loads(line)
        assert e["case"] not in out, f"duplicate fixture {e['case']}"
        out[e["case"]] = e
    return out


def test_exact_join_fixtures_reproduce_par_bitmap_pairs():
    g = load()
    a, b = g["C3"], g["C3_exact"]
    assert a["collection_sha256"] == b["collection_sha256"]
    assert a["pair_count"] == b["pair_count"] == 203594341
    assert a["pairs_sha256"] == b["pairs_sha256"]


def test_every_heavy_config_has_full_size_pairs():
    g = load()
    for case, n in (("C4_exact", 42380999), ("C5_exact", 60633248)):
        assert g[case]["pair_count"] == n
        assert len(g[case]["pairs_sha256"]) == 64 and len(g[case]["collection_sha256"]) == 64
