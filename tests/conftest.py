import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("MKL_NUM_THREADS", "1")

GOLDEN = os.path.join(ROOT, "tests", "golden")
SEED = 20250814


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def rel(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def configs32():
    return ["".join("s" if (bits >> (4 - i)) & 1 else "d" for i in range(5)) for bits in range(32)]


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import orc as _orc

    return _orc()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import have_ref, ref as _ref

    if not have_ref():
        pytest.skip("oracle/_ref (the compiled reference) is not built here")
    return _ref()


def make_inputs(chk, nm, nd, nt, fill="uni", seed=SEED):
    if fill == "uni":
        f = lambda n, k: chk.uniform_fill(n, chk.seed_stream(seed, k))  # noqa: E731
    else:
        f = lambda n, k: chk.non_representable_fill(n, chk.seed_stream(seed, k))  # noqa: E731
    return f(nm * nd * nt, 0), f(nm * nt, 1), f(nd * nt, 2)
