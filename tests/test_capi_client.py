"""The reference's own C client test, proj/tests/test_capi.cpp, compiled
UNCHANGED against the B200 library (oracle/Makefile -> oracle/_ref/test_capi_b200,
built in the container that holds the reference sources; the binary travels
to the GPU box).  It drives the ABI the way an external C client does: option
structs, opaque handles, status codes, error strings -- and joins the same
collection with NAIVE, ALLPAIRS, PPJOIN, PPJOIN+, GROUPJOIN, ADAPTJOIN and
PAR_BITMAP, requiring byte-identical pair lists (test_capi.cpp:64-88)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "test_capi_b200")
LIB = os.path.join(ROOT, "paper_1711_07295_b200", "lib", "libssjoin.so")


def _need_bin():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_capi_b200 not built (reference sources absent)")


def test_reference_client_links_the_product_library():
    _need_bin()
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True, check=True).stdout
    line = [x for x in out.splitlines() if "libssjoin.so" in x]
    assert line and os.path.realpath(line[0].split("=>")[1].split()[0]) == os.path.realpath(LIB), out


@pytest.mark.gpu
def test_reference_client_passes(tmp_path):
    _need_bin()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600, env=dict(os.environ, TMPDIR=str(tmp_path)))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all checks passed" in r.stdout
