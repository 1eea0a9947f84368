"""Lattice-aligned poses on every query path.

A rotation whose column a has a single nonzero entry (the 24 cube
rotations, or any screw about a grid axis) puts the reference index u_a of
EVERY mode on an integer, so every mode takes the float64 tie decision
(_core.pyx:633-643).  The kernels serve those axes from a per-pose tie table
(cascade_single.cu, cascade.cu, field.cu); these tests pin that table to the
oracle on the single-query kernel, the resident server, the batched sweep
and the landscape, at the stated tolerances (fp32 1e-4, fp64 1e-10 of
max(|ref|, L1) for queries; landscapes relative to max |ref|).
"""

import numpy as np
import pytest

import oracle
from conftest import lattice_rotations_3d, parity_tol, synthetic_window

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "fp64": 1e-10}


def axis_rotation(axis, angle):
    c, s = np.cos(angle), np.sin(angle)
    i, j = [(1, 2), (2, 0), (0, 1)][axis]
    R = np.eye(3)
    R[i, i], R[i, j], R[j, i], R[j, j] = c, -s, s, c
    return R


def aligned_poses(rng):
    rots = list(lattice_rotations_3d())
    rots += [axis_rotation(a, rng.uniform(0, 2 * np.pi)) for a in (0, 1, 2) for _ in range(2)]
    rots.append(axis_rotation(2, np.pi / 2) @ axis_rotation(0, 0.4))  # one aligned column only
    return rots


@pytest.fixture(scope="module")
def be():
    from paper_1711_05017_b200 import backend

    return backend


@pytest.mark.parametrize("wrap", [False, True])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_single_and_batch_match_oracle(be, wrap, prec):
    import torch

    rng = np.random.default_rng(21)
    w = 12
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom = (1.0 / (16 * 0.3), 1.0 / (16 * 0.3), 1.0 / (16 * 0.3))  # non-dyadic: ties on both sides
    centre = np.array([0.1, -0.2, 0.3])
    Rs = aligned_poses(rng)
    ts = rng.uniform(-1, 1, size=(len(Rs), 3))
    poses = torch.from_numpy(be.pack_poses(np.stack(Rs), ts)).cuda()
    batch = be.cascade_batch(W1, W2, wrap, dom, 0.5, centre, poses, precision=prec).cpu().numpy().view(np.complex128)
    for i, (R, t) in enumerate(zip(Rs, ts)):
        want = oracle.cascade(C1, C2, wrap, dom, 0.5, R, t, centre)
        l1 = oracle.cascade_term_scales(C1, C2, wrap, dom, 0.5, R, t, centre)
        single = be.cascade(W1, W2, wrap, dom, 0.5, R, t, centre, precision=prec)
        assert np.all(parity_tol(single, want, l1, TOL[prec])), (i, single, want)
        assert np.all(parity_tol(batch[i], want, l1, TOL[prec])), (i, batch[i], want)


def test_server_matches_oracle(be):
    rng = np.random.default_rng(22)
    w = 16
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom = (1.0 / (16 * 0.3),) * 3
    centre = np.array([0.2, 0.1, -0.1])
    with be.HapticServer(W1, W2, False, dom, 0.5, centre, "fp32"):
        for R in aligned_poses(rng)[::2]:
            t = rng.uniform(-1, 1, size=3)
            got = be.cascade(W1, W2, False, dom, 0.5, R, t, centre, precision="fp32")
            want = oracle.cascade(C1, C2, False, dom, 0.5, R, t, centre)
            l1 = oracle.cascade_term_scales(C1, C2, False, dom, 0.5, R, t, centre)
            assert np.all(parity_tol(got, want, l1, TOL["fp32"]))


@pytest.mark.parametrize("w", [None, 8])
@pytest.mark.parametrize("precision,rtol", [(64, 1e-10), (32, 2e-5)])
def test_landscape_matches_oracle(be, w, precision, rtol):
    from paper_1711_05017_b200.descriptor import SampleGrid
    from paper_1711_05017_b200.energy import score_field_device

    rng = np.random.default_rng(23)
    N, h = 16, 0.3
    dims, origin = (N,) * 3, (-0.5 * N * h + 0.5 * h,) * 3
    g = SampleGrid(3, dims, origin, h)
    side = N if w is None else w
    C1, C2 = synthetic_window(rng, side), synthetic_window(rng, side)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)

    class Part:
        def __init__(self, win):
            self.grid, self.win = g, win

        def window(self, m_prime=None):
            return self.win, w is None

    for R in (np.eye(3), lattice_rotations_3d()[5], axis_rotation(1, 0.9)):
        got = score_field_device(Part(W1), Part(W2), R, None, precision=precision).cpu().numpy()
        want = oracle.score_field(C1, C2, w is None, dims, origin, h, R).ravel()
        np.testing.assert_allclose(got, want, rtol=0, atol=rtol * np.max(np.abs(want)))
