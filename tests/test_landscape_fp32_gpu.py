"""The fp32 landscape (complex64 windows: product kernel + three FFT passes,
gf_score_field) against the float64 path (pinned to the oracle by
test_spectral_gpu / test_baseline_parity_gpu), across pose kinds (random,
identity, lattice rotations through the tie tables, screws), truncated and
full spectra, at the BASELINE tolerance |new - ref| <= 1e-4 max(|ref|, L1)."""

import numpy as np
import pytest

import oracle
from conftest import random_rotation
from paper_1711_05017_b200 import backend as be
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.energy import score_field_device

pytestmark = pytest.mark.gpu


class _Pair:
    def __init__(self, grid, win, wrap):
        self.grid, self._w = grid, (win, wrap)

    def window(self, m_prime=None):
        return self._w


def _rot(axis, ang):
    c, s = np.cos(ang), np.sin(ang)
    R = np.eye(3)
    i, j = [(1, 2), (0, 2), (0, 1)][axis]
    R[i, i], R[i, j], R[j, i], R[j, j] = c, -s, s, c
    return R


def _window(rng, w):
    k2 = (np.arange(w) - w // 2).astype(np.float64) ** 2
    amp = 1.0 / (1.0 + k2[:, None, None] + k2[None, :, None] + k2[None, None, :])
    return (rng.standard_normal((w,) * 3) + 1j * rng.standard_normal((w,) * 3)) * amp


POSES = {
    "random": lambda rng: random_rotation(rng),
    "identity": lambda rng: np.eye(3),
    "z90": lambda rng: _rot(2, np.pi / 2),           # lattice: tie tables on every axis
    "x_to_z": lambda rng: _rot(1, np.pi / 2 - 0.2),  # mode x nearly along C2's z
    "screw": lambda rng: _rot(2, 0.7),               # one lattice-aligned axis (the C5 trajectory)
}


@pytest.mark.parametrize("n,w", [(64, 64), (64, 32), (128, 128), (128, 96), (256, 64)])
@pytest.mark.parametrize("pose", sorted(POSES))
def test_fp32_landscape_matches_fp64_path(n, w, pose):
    rng = np.random.default_rng(n * 1000 + w + len(pose))
    h = 3.0 / n
    g = SampleGrid(3, (n,) * 3, (-1.5,) * 3, h)
    C1, C2 = _window(rng, w), _window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    wrap = w == n
    R = POSES[pose](rng)
    a1, a2 = _Pair(g, W1, wrap), _Pair(g, W2, wrap)
    got = score_field_device(a1, a2, R, None, precision=32).cpu().numpy().astype(np.complex128)
    ref = score_field_device(a1, a2, R, None, precision=64).cpu().numpy()
    l1 = oracle.score_field_scale(C1, C2, wrap, g.dims, h, R)
    err = np.abs(got - ref)
    assert np.all(err <= 1e-4 * np.maximum(np.abs(ref), l1)), float(np.max(err / np.maximum(np.abs(ref), l1)))


def test_fp32_landscape_deterministic():
    rng = np.random.default_rng(7)
    n = 128
    g = SampleGrid(3, (n,) * 3, (-1.0,) * 3, 2.0 / n)
    W1, W2 = be.DeviceWindow(_window(rng, n)), be.DeviceWindow(_window(rng, n))
    R = random_rotation(rng)
    a = score_field_device(_Pair(g, W1, True), _Pair(g, W2, True), R, None, precision=32)
    b = score_field_device(_Pair(g, W1, True), _Pair(g, W2, True), R, None, precision=32)
    assert bool((a == b).all())
