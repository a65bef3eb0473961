import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "blockmv_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def pytest_collection_modifyitems(config, items):
    """Skip GPU-marked tests on a host without a CUDA device (instead of
    failing them with a driver error)."""
    if has_cuda():
        return
    skip = pytest.mark.skip(reason="needs a CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["__meta__"]).decode())
    return z, meta


def checksum(a) -> float:
    """Same fingerprint as tests/golden/make_golden.py."""
    a = np.asarray(a)
    return float(np.sum(np.abs(a.astype(np.complex128)) * np.arange(1, a.size + 1) % 7.0))


def golden_inputs(p):
    """Regenerate a golden case's (flat A, ld, x, y) from its seed and check
    the fingerprints recorded by make_golden.py."""
    from oracle import naive

    rng = np.random.default_rng(p["seed"])
    flat, ld = naive.random_matrix(rng, p["rows"], p["cols"], p["tag"])
    x = naive.random_vec(rng, p["xl"], p["tag"])
    y = naive.random_vec(rng, p["yl"], p["tag"])
    assert ld == p["ld"]
    assert abs(checksum(flat) - p["sum_A"]) <= 1e-9 * max(1.0, abs(p["sum_A"]))
    assert abs(checksum(x) - p["sum_x"]) <= 1e-9 * max(1.0, abs(p["sum_x"]))
    assert abs(checksum(y) - p["sum_y"]) <= 1e-9 * max(1.0, abs(p["sum_y"]))
    return flat, ld, x, y


def cfg1_inputs(n=4096):
    """BASELINE config 1 inputs by the cli.py recipe (cli.py:52-57,100-125)."""
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, size=(n, n)).astype(np.float64)
    x = rng.uniform(-1, 1, size=n).astype(np.float64)
    y = rng.uniform(-1, 1, size=n).astype(np.float64)
    return np.asfortranarray(a), x, y


@pytest.fixture(scope="session")
def golden():
    return load_golden()


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
