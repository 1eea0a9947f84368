"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)

SEED = 20260814  # the reference suite's seed (pkg/tests/conftest.py:14)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture
def rng():
    return np.random.default_rng(SEED)


def lattice_rotations_3d():
    """The 24 proper rotations of the cube (reference conftest.py:40-53)."""
    from itertools import permutations

    out = []
    for perm in permutations(range(3)):
        for signs in np.ndindex(2, 2, 2):
            R = np.zeros((3, 3))
            for row, col in enumerate(perm):
                R[row, col] = -1.0 if signs[row] else 1.0
            if np.linalg.det(R) > 0.5:
                out.append(R)
    return out


def random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def synthetic_window(rng, w, d=3):
    """CN(0,1) (1+|k|^2)^-1 window (SURVEY.md 8(d) micro-benchmark distribution)."""
    shape = (w,) * d
    k = np.stack(np.meshgrid(*[np.arange(w) - w // 2] * d, indexing="ij"), axis=-1)
    amp = 1.0 / (1.0 + np.sum(k * k, axis=-1))
    z = rng.normal(size=shape) + 1j * rng.normal(size=shape)
    return z * amp


def parity_tol(got, want, l1, rel):
    """|got - want| <= rel * max(|want|, L1)."""
    return np.abs(got - want) <= rel * np.maximum(np.abs(want), l1)
