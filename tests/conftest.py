import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200, sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def rng():
    return np.random.default_rng(0)


def random_signs(rng, rows, cols):
    """pkg/tests/conftest.py:7-8"""
    return rng.integers(0, 2, size=(rows, cols)).astype(np.float64) * 2.0 - 1.0


def f32_vector(rng, size, positive=False):
    """pkg/tests/conftest.py:11-14"""
    vals = rng.standard_normal(size).astype(np.float32).astype(np.float64)
    return np.abs(vals) + 0.1 if positive else vals


def rel_norm(out, ref):
    return float(np.linalg.norm(np.asarray(out) - ref) / max(np.linalg.norm(ref), 1e-300))


def rel_max(out, ref):
    return float(np.max(np.abs(np.asarray(out) - ref)) / max(np.max(np.abs(ref)), 1e-300))


def random_layer(rng, n, k, m, positive=False):
    """pkg/tests/conftest.py:17-24 (GPU pack)"""
    from paper_2505_11076_b200 import DbfLayer, pack

    return DbfLayer(
        a=f32_vector(rng, n, positive),
        A=pack(random_signs(rng, n, k)),
        mid=f32_vector(rng, k, positive),
        B=pack(random_signs(rng, k, m)),
        b=f32_vector(rng, m, positive),
    )
