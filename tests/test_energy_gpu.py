"""Stage 3 through the public API: evaluate / score_at / gradients on assets
built entirely on the GPU, vs the reference's golden evaluations, in fp64
(1e-9) and fp32 (1e-4 of max(|ref|, L1) -- BASELINE.md section 2)."""

import os

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import backend, scenes
from paper_1711_05017_b200.descriptor import KernelSpec, affinity_field, indicator_field
from paper_1711_05017_b200.energy import (Configuration, PartAsset, evaluate, rotational_gradient, score_at,
                                          translational_gradient)

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_small.npz"))


@pytest.fixture(scope="module")
def peg_assets():
    peg = scenes.get_scene("peg3d")
    g = peg.grid(16)
    f1 = affinity_field(peg.fixed, g, KernelSpec())
    f2 = affinity_field(peg.moving, g, KernelSpec())
    a1 = PartAsset.from_field("fixed", f1, solid_box=peg.fixed.bbox)
    a2 = PartAsset.from_field("moving", f2, movable=True, solid_box=peg.moving.bbox)
    return a1, a2


@pytest.mark.parametrize("prec,rtol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_evaluate_matches_reference_golden(peg_assets, prec, rtol):
    a1, a2 = peg_assets
    prev = backend.precision()
    backend.set_precision(prec)
    try:
        for pose, want in zip(GOLD["eval3d_poses"], GOLD["eval3d_results"]):
            R, t, mp = pose[:9].reshape(3, 3), pose[9:12], int(pose[12])
            res = evaluate(a1, a2, Configuration(R, t), mp or None)
            got = np.concatenate([[res.score.real, res.score.imag], res.force, res.torque])
            assert res.energy == -res.score.real
            assert res.modes_used == (mp or 4096)
            np.testing.assert_allclose(got, want, rtol=rtol, atol=rtol * np.max(np.abs(want)))
    finally:
        backend.set_precision(prev)


def test_score_matches_brute_at_lattice_rotations():
    """Indicator pair, lattice rotations, node translations: the cascade is
    the exact real-space overlap sum (reference test_energy.py:111-122)."""
    fixed = scenes.box_mesh((1.2, 0.8, 0.6))
    moving = scenes.box_mesh((0.5, 0.5, 0.9))
    grid = scenes.grid_for_pair(fixed, moving, 16)
    f1, f2 = indicator_field(fixed, grid), indicator_field(moving, grid)
    a1 = PartAsset.from_field("fixed", f1, solid_box=fixed.bbox)
    a2 = PartAsset.from_field("moving", f2, movable=True, solid_box=moving.bbox)
    backend.set_precision("fp64")
    try:
        from conftest import lattice_rotations_3d

        for R in [lattice_rotations_3d()[k] for k in (0, 7, 16, 23)]:
            for t in ([0.0, 0.0, 0.0], [grid.spacing, -2 * grid.spacing, 0.0]):
                got = score_at(a1, a2, Configuration(R, t))
                P = grid.points()
                Q = (P - np.asarray(t)) @ R
                u = (Q - np.asarray(grid.origin)) / grid.spacing
                idx = np.rint(u).astype(int)
                ok = np.all((idx >= 0) & (idx < 16), axis=1)
                v2 = np.zeros(len(P))
                v2[ok] = f2.values.real.reshape(grid.dims)[tuple(idx[ok].T)]
                want = np.sum(f1.values.real * v2) * grid.cell_volume
                assert got == pytest.approx(want, rel=1e-9, abs=1e-12)
    finally:
        backend.set_precision("fp32")


def test_gradients_match_finite_differences(peg_assets):
    a1, a2 = peg_assets
    backend.set_precision("fp64")
    try:
        R = oracle.quat_rotation([0.95, 0.1, 0.2, -0.15])
        t = np.array([0.2, -0.1, 0.15])
        cfg = Configuration(R, t)
        tg = translational_gradient(a1, a2, cfg, 512)
        eps = 1e-6
        for a in range(3):
            e = np.zeros(3)
            e[a] = eps
            fd = (score_at(a1, a2, Configuration(R, t + e), 512) - score_at(a1, a2, Configuration(R, t - e), 512)) / (
                2 * eps)
            assert abs(tg[a] - fd) <= 1e-5 * max(abs(fd), 1e-9) + 1e-9
        rg = rotational_gradient(a1, a2, cfg, 512)
        assert rg.shape == (3,)
        vec = rotational_gradient(a1, a2, cfg, None, path="vector")
        assert vec.shape == (3,)
        with pytest.raises(ValueError):
            rotational_gradient(a1, a2, cfg, path="nope")
    finally:
        backend.set_precision("fp32")


@pytest.mark.parametrize("d,m_prime", [(3, None), (3, 512), (2, None)])
def test_vector_path_torque_matches_restatement(d, m_prime):
    """The moment-spectrum torque (gf_vector_torque: one fused float64 pass)
    against the numpy restatement of energy.py:210-251 on the same windows,
    in 3D (full and truncated) and 2D."""
    import oracle
    from paper_1711_05017_b200 import scenes
    from paper_1711_05017_b200.descriptor import KernelSpec, affinity_field

    sc = scenes.get_scene("peg3d" if d == 3 else "peg2d")
    g = sc.grid(16 if d == 3 else 32)
    a1 = PartAsset.from_field("f", affinity_field(sc.fixed, g, KernelSpec()), solid_box=sc.fixed.bbox)
    a2 = PartAsset.from_field("m", affinity_field(sc.moving, g, KernelSpec()), movable=True,
                              solid_box=sc.moving.bbox)
    rng = np.random.default_rng(40 + d)
    (w1, wrap1), (w2, wrap2) = a1.window(m_prime), a2.window(m_prime)
    moments = [np.asarray(mw) for mw in a2.moment_window(m_prime)]
    c, dom, dcell = g.center(), g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
    for _ in range(3):
        if d == 3:
            q = rng.normal(size=4)
            R = oracle.quat_rotation(q)
        else:
            th = rng.uniform(0, 2 * np.pi)
            R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        t = rng.uniform(-0.3, 0.3, d)
        got = rotational_gradient(a1, a2, Configuration(R, t), m_prime, path="vector")
        want = oracle.rotational_gradient_vector(np.asarray(w1), np.asarray(w2), moments, wrap1 and wrap2, dom,
                                                 dcell, R, t, c)
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-12 * np.max(np.abs(want)))
