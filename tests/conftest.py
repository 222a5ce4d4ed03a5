import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def port():
    from oracle import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    from oracle import Ref, build_ref
    if build_ref() is None:
        pytest.skip("reference library (oracle/_ref) not built on this machine")
    return Ref()


def _load(name):
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def kat():
    return _load("kat_reference.npz")


@pytest.fixture(scope="session")
def material_kat():
    return _load("material.npz")


@pytest.fixture(scope="session")
def runs_kat():
    return _load("runs.npz")
