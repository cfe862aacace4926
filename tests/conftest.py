"""Shared fixtures. GPU tests are marked ``gpu`` and never skip silently on a GPU box:
a missing library or CUDA device there is a failure, not a fallback."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def port():
    import oracle
    if not oracle.available("port"):
        oracle.build("port")
    return oracle.load("port")


@pytest.fixture(scope="session")
def checker():
    """The strongest CPU oracle present: the compiled reference, else the C port."""
    import oracle
    if not oracle.available("port"):
        oracle.build("port")
    return oracle.load("best")


@pytest.fixture(scope="session")
def reference():
    import oracle
    if not oracle.available("reference"):
        pytest.skip("compiled reference (oracle/_ref) not present")
    return oracle.load("reference")


@pytest.fixture(scope="session")
def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as f:
        return json.load(f)


def load_case(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def p3s():
    import paper_2009_09501_b200 as m
    if not os.path.exists(m.LIB_PATH):
        m.build()
    m.lib()
    return m
