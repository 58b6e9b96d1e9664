"""Shared fixtures.  ``gpu``-marked tests need a B200; everything else runs
on CPU (the driver runs ``-m "not gpu"`` in the build container)."""
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
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def random_euclidean_matrix(n, rng):
    """Restates the reference fixture (pkg/tests/conftest.py:27-31)."""
    pts = rng.random((n, 2)) * 10.0
    c = np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))
    np.fill_diagonal(c, 0.0)
    return c


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def golden_matrix(golden, inst):
    if inst.startswith("euclid"):
        _, n, s = inst.split(":")
        return random_euclidean_matrix(int(n), np.random.default_rng(int(s)))
    return np.array(golden["matrices"][inst], dtype=float)


def golden_params(golden, case):
    p = dict(case["params"])
    if p.get("seed_tour") == "boustrophedon":
        p["seed_tour"] = golden["seed_tours"][case["instance"]]
    return p


@pytest.fixture(scope="session")
def golden_e2e():
    return load_golden("golden_e2e.json")


@pytest.fixture(scope="session")
def golden_kernels():
    return load_golden("golden_kernels.json")


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
