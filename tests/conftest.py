import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


PY_CASES = ["smoke", "unclamped", "m16", "n1m8", "m1"]
ALL_CASES = PY_CASES + ["accept_small"]


def load_golden(name):
    """(npz dict, index path, model path or None)"""
    z = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    model = os.path.join(GOLDEN, f"{name}.model.vlq")
    return z, os.path.join(GOLDEN, f"{name}.index.vlq"), (model if os.path.exists(model) else None)


def grid_of(z):
    return [(int(w1), float(np.float32(a)), int(k)) for w1, a, k in z["grid"]]


def regen_base(z):
    """Regenerates the fixture's base set with the engine's bit-identical
    gen_synthetic (dataset.cpp:13-44) and checks it against the stored head."""
    from paper_1901_00275_b200 import vlqadc
    count, dim, clusters, spread, seed = z["base_params"]
    base = vlqadc.gen_synthetic(int(count), int(dim), clusters=int(clusters), spread=float(spread), seed=int(seed))
    assert np.array_equal(base[:64], z["base_head"])
    return base


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle
    return oracle
