"""B200-native Bitmap-Filter set-similarity self-join (arXiv 1711.07295, Alg. 8).

The product is the C-ABI shared library ``lib/libssjoin.so`` built from
``csrc/`` (host C++ + sm_100a CUDA kernels); it is a drop-in for the
reference engine's ``libssjoin`` (``include/ssjoin.h``).  This package only
locates and binds it; :mod:`.ssjoin` mirrors the reference's C interface in
Python.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

from . import capi

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# SSJB_LIB points experiments at another build of the same library (A/B timing)
LIB_PATH = os.environ.get("SSJB_LIB") or os.path.join(PKG_DIR, "lib", "libssjoin.so")
CSRC_DIR = os.path.join(PKG_DIR, "csrc")

_lib = None


def build(jobs: int = 8) -> str:
    """Compile libssjoin.so in-tree (nvcc for sm_100a; runs without a GPU)."""
    subprocess.run(["make", "-s", "-C", CSRC_DIR, f"-j{jobs}"], check=True)
    return LIB_PATH


def load_library() -> ctypes.CDLL:
    """The B200 library.  Raises if it has not been built: there is no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -c 'import __graft_entry__ as g; g.build()'` "
                               "or `make -C paper_1711_07295_b200/csrc`")
        _lib = capi.bind(ctypes.CDLL(LIB_PATH), extensions=True)
    return _lib
