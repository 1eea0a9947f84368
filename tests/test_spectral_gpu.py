"""Stage 2 (forward DFT, truncation, centred window, inverse) and stage 4
(landscape, rotate/reflect) on the GPU vs the oracle and golden fixtures.
float64 engine: 1e-12 of the spectrum scale."""

import os

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import scenes
from paper_1711_05017_b200.descriptor import ComplexField, KernelSpec, SampleGrid, affinity_field
from paper_1711_05017_b200.energy import PartAsset, score_field
from paper_1711_05017_b200.spectral import (center_window, forward_dft, forward_window, inverse_dft,
                                            rotate_reflect_spectrum, truncate)

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_small.npz"))


def random_field(rng, dims, origin, h):
    g = SampleGrid(len(dims), dims, origin, h)
    v = rng.normal(size=g.node_count) + 1j * rng.normal(size=g.node_count)
    return ComplexField(g, v)


@pytest.mark.parametrize("dims", [(16, 16, 16), (8, 32, 16), (64, 64), (32, 64, 128)])
def test_forward_inverse_dft(dims):
    rng = np.random.default_rng(len(dims) + dims[0])
    origin = tuple(-0.37 * n * 0.05 for n in dims)
    f = random_field(rng, dims, origin, 0.05)
    A = forward_dft(f)
    want = oracle.forward_dft(f.values, dims, origin, 0.05)
    np.testing.assert_allclose(A.amplitudes.reshape(dims), want, atol=1e-12 * np.max(np.abs(want)))
    back = inverse_dft(A)
    np.testing.assert_allclose(back.values, f.values, atol=1e-12 * np.max(np.abs(f.values)))


def test_windows_match_reference_golden():
    peg = scenes.get_scene("peg3d")
    g = peg.grid(16)
    f1 = affinity_field(peg.fixed, g, KernelSpec())
    s1 = forward_dft(f1)
    scale = np.max(np.abs(GOLD["spec3d_fixed_full"]))
    np.testing.assert_allclose(s1.amplitudes, GOLD["spec3d_fixed_full"], atol=1e-12 * scale)
    np.testing.assert_allclose(center_window(truncate(s1, 512)), GOLD["win3d_fixed_m512"], atol=1e-12 * scale)
    np.testing.assert_allclose(center_window(s1), GOLD["win3d_fixed_full"], atol=1e-12 * scale)
    # the pruned direct path field -> centred window
    np.testing.assert_allclose(forward_window(f1, 8).cpu().numpy(), GOLD["win3d_fixed_m512"], atol=1e-12 * scale)


def test_score_field_matches_reference_golden():
    peg = scenes.get_scene("peg3d")
    g = peg.grid(16)
    f1 = affinity_field(peg.fixed, g, KernelSpec())
    f2 = affinity_field(peg.moving, g, KernelSpec())
    a1 = PartAsset.from_field("fixed", f1, solid_box=peg.fixed.bbox)
    a2 = PartAsset.from_field("moving", f2, movable=True, solid_box=peg.moving.bbox)
    R = GOLD["field3d_R"]
    for mp, key in ((512, "field3d_m512"), (None, "field3d_full")):
        land = score_field(a1, a2, R, mp)
        want = GOLD[key]
        np.testing.assert_allclose(land.values, want, atol=1e-11 * np.max(np.abs(want)))
    np.testing.assert_array_equal(land.wrap_mask.ravel(), GOLD["field3d_wrap_mask"])


def test_score_field_2d_and_noncubic_vs_oracle():
    rng = np.random.default_rng(5)
    for dims, w in (((32, 32), 16), ((32, 32), None), ((16, 32, 32), None)):
        h = 0.1
        origin = tuple(-0.5 * n * h for n in dims)
        f1, f2 = random_field(rng, dims, origin, h), random_field(rng, dims, origin, h)
        a1 = PartAsset.from_field("a", f1)
        a2 = PartAsset.from_field("b", f2, movable=True)
        d = len(dims)
        if d == 2:
            th = 0.37
            R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        else:
            R = oracle.quat_rotation([0.8, 0.3, -0.2, 0.1])
        mp = None if w is None else w ** d
        land = score_field(a1, a2, R, mp).values
        A1 = oracle.forward_dft(f1.values, dims, origin, h)
        A2 = oracle.forward_dft(f2.values, dims, origin, h)
        C1 = oracle.center_window(A1, dims, origin, h, w)
        C2 = oracle.center_window(A2, dims, origin, h, w)
        want = oracle.score_field(C1, C2, w is None, dims, origin, h, R).ravel()
        np.testing.assert_allclose(land, want, atol=1e-10 * np.max(np.abs(want)))


def test_rotate_reflect_identity_is_negation():
    rng = np.random.default_rng(9)
    dims, h = (16, 16, 16), 0.1
    f = random_field(rng, dims, tuple(-0.8 for _ in dims), h)
    s = truncate(forward_dft(f), 8 ** 3)
    out = rotate_reflect_spectrum(s, np.eye(3)).reshaped()
    win = s.reshaped()
    # A(-w): index negation inside the window; the k = -w/2 plane maps outside (zero)
    want = np.zeros_like(win)
    want[1:, 1:, 1:] = win[1:, 1:, 1:][::-1, ::-1, ::-1]
    np.testing.assert_allclose(out, want, atol=1e-12 * np.max(np.abs(win)))


@pytest.mark.parametrize("N,w,prec", [((64, 32, 64), 16, 64), ((128, 128, 64), 32, 32)])
def test_forward_window_node_slabs_bit_identical(N, w, prec):
    """Multi-GPU W1 path: inner passes per rank's x-planes, the all-to-all's
    re-slicing (done here in-process), the x pass per window y-slab -- equal,
    bit for bit, to the single-GPU forward_window."""
    import torch

    from paper_1711_05017_b200 import parallel
    from paper_1711_05017_b200.spectral import _fft3

    rng = np.random.default_rng(7)
    f = random_field(rng, N, tuple(-0.5 * n * 0.02 for n in N), 0.02)
    g = f.grid
    dt = torch.complex128 if prec == 64 else torch.complex64
    x = f.device_values().reshape(N).to(dt)
    want = _fft3(x, (w,) * 3, -1, False, True, [0.0] * 3, [0.5] * 3, g.cell_volume, precision=prec)
    for world in (2, 3):
        x_r = [parallel.shard_range(N[0], r, world) for r in range(world)]
        wy_r = [parallel.shard_range(w, r, world) for r in range(world)]
        inner = [parallel.window_inner_passes(x[lo:hi].contiguous(), N, w, prec) for lo, hi in x_r]
        outs = []
        for ylo, yhi in wy_r:
            slab = torch.cat([b[:, ylo:yhi] for b in inner], dim=0).contiguous()
            outs.append(parallel.window_outer_pass(slab, N, w, g.cell_volume, prec))
        got = torch.cat(outs, dim=1)
        assert torch.equal(got, want)
        # fused variant: each rank's y pass stores into every rank's window y-slab
        slabs = [torch.zeros((N[0], hi - lo, w), dtype=dt, device="cuda") for lo, hi in wy_r]
        bounds = [lo for lo, _ in wy_r] + [wy_r[-1][1]]
        for lo, hi in x_r:
            a = parallel._wpass(x[lo:hi].contiguous(), (hi - lo, N[1], w), 2, N[2], 1.0, prec)
            parallel.scatter_y_pass(a, N[1], bounds, [t.data_ptr() for t in slabs], lo, prec, forward=True)
        fused = torch.cat([parallel.window_outer_pass(sl, N, w, g.cell_volume, prec) for sl in slabs], dim=1)
        assert torch.equal(fused, want)
    # world 1 through the public entry (no process group)
    assert torch.equal(parallel.forward_window_slab(x, g, w, precision=prec), want)
