import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running sweep")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_regression():
    return _load_json("regression.json")


@pytest.fixture(scope="session")
def golden_streams():
    return _load_json("streams.json")


@pytest.fixture(scope="session")
def golden_meta():
    return _load_json("vectors.json")


@pytest.fixture(scope="session")
def golden_vectors():
    with np.load(os.path.join(GOLDEN, "vectors.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_census():
    return _load_json("census.json")


@pytest.fixture(scope="session")
def golden_derive_all():
    return _load_json("derive_all.json")


@pytest.fixture(scope="session")
def oracle_stream0(golden_regression):
    from oracle import rsa_oracle as O
    return O.from_fields(golden_regression["params"])


@pytest.fixture(scope="session")
def census_c():
    """(sorted safe primes of [2^31, 2^32), prime count) from the C oracle."""
    from oracle import coracle
    return coracle.census()
