import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_arrays():
    return np.load(os.path.join(GOLDEN_DIR, "golden_pairs.npz"))


@pytest.fixture(scope="session")
def lib():
    """The B200 product library (built in-tree)."""
    from paper_1711_07295_b200 import load_library
    return load_library()


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def ref():
    """The reference compiled from its sources (oracle/_ref); skipped when absent."""
    from oracle import oracle as O
    r = O.ref_lib()
    if r is None:
        pytest.skip("oracle/_ref/libssjoin_ref.so not built (reference sources absent)")
    return r


def golden_collection(golden_arrays, name):
    return (golden_arrays[f"coll/{name}/tokens"], golden_arrays[f"coll/{name}/offsets"])


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
