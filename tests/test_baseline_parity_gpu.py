"""Parity at the BASELINE.json configurations' own sizes.

* C2 (128^3, K=32: w = 64, truncated) -- the headline query, on synthetic
  windows and on the GPU-built low-clearance peg-in-hole assets through
  evaluate(), against the reference's compiled kernel (oracle/_ref,
  _core.pyx:598-724) when it is built and the C restatement otherwise;
* C5 (256^3, K=64: w = 128) -- generic poses and the screw trajectory's
  z-axis rotations (a lattice-aligned axis: the per-pose tie tables);
* C3 (256^3, K=48: w = 96) -- the batched sweep on cmd_bench poses
  (cli.py:336-346);
* C4 -- the landscape (energy.py:309-344) at 256^3 with the full spectrum
  against the numpy restatement of score_field, and at 512^3 (full spectrum
  and an m' = 128^3 window) on sampled voxels against the C restatement of
  the cascade: landscape[j] = score_at(t = p_j);
* D -- affinity_field (descriptor.py:309-357) at 64^3 on the peg-in-hole
  meshes and at 32^3 on the gear-pair and bolt-nut meshes: flags, excluded,
  inside and the stats bit for bit, values to 1e-12.

Tolerances: fp32 |new - ref| <= 1e-4 max(|ref|, L1),
L1 = dcell sum |summand|; fp64 1e-10 (query) / 1e-9 (landscape).  The plain
relative error max|new - ref| / max|ref| is asserted too where it is
meaningful (fp64: 1e-9; fp32 queries: 1e-3).
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from conftest import parity_tol, random_rotation
from paper_1711_05017_b200 import backend as be
from paper_1711_05017_b200 import scenes
from paper_1711_05017_b200.descriptor import SampleGrid, affinity_field
from paper_1711_05017_b200.energy import Configuration, evaluate, score_field_device

pytestmark = pytest.mark.gpu

# config -> (grid N, grid_for_pair domain, window side w)
CONFIGS = {"C2": (128, 3.46, 64), "C3": (256, 5.42, 96), "C5": (256, 4.37, 128)}


def lean_window(rng, w):
    """CN(0,1)(1+|k|^2)^-1 without an (w^3, 3) index array."""
    k2 = (np.arange(w) - w // 2).astype(np.float64) ** 2
    amp = 1.0 / (1.0 + k2[:, None, None] + k2[None, :, None] + k2[None, None, :])
    z = rng.standard_normal((w, w, w)) + 1j * rng.standard_normal((w, w, w))
    z *= amp
    return z


def grid_consts(n, domain):
    h = domain / n
    origin = -0.5 * domain
    c = np.full(3, origin + h * (n // 2))
    return h, origin, c, np.full(3, 1.0 / (n * h)), 1.0 / (n ** 3 * h ** 3)


def reference_cascade(C1, C2, wrap, dom, dcell, R, t_eff, c):
    """The reference's own compiled kernel when oracle/_ref is built (the
    oracle restatement is then also pinned against it at this size)."""
    want = oracle.cascade(C1, C2, wrap, dom, dcell, R, t_eff, c)
    core = oracle.ref_core()
    if core is not None:
        ref = core.cascade_3d(C1, C2, bool(wrap), *dom, dcell, np.ascontiguousarray(R), np.ascontiguousarray(t_eff),
                              np.ascontiguousarray(c))
        np.testing.assert_allclose(want, ref, rtol=0, atol=1e-12 * np.max(np.abs(ref)))
        return np.asarray(ref)
    return want


def poses_for(kind, rng, n, domain, c):
    Rs, ts = [], []
    if kind == "generic":
        for _ in range(n):
            Rs.append(random_rotation(rng))
            ts.append(rng.uniform(-0.25 * domain, 0.25 * domain, 3))
    else:  # the C5 screw: R_z(theta), t_z = 0.3 - pitch theta / 2 pi (pitch 0.1); lattice angles included
        for th in (0.0, 0.5 * np.pi, 0.3, 2.5, 5.9)[:n]:
            cth, sth = np.cos(th), np.sin(th)
            Rs.append(np.array([[cth, -sth, 0.0], [sth, cth, 0.0], [0.0, 0.0, 1.0]]))
            ts.append(np.array([0.0, 0.0, 0.3 - 0.1 * th / (2 * np.pi)]))
    return [(R, t - c + R @ c) for R, t in zip(Rs, ts)]


@pytest.mark.parametrize("cfg", ["C2", "C5"])
@pytest.mark.parametrize("kind", ["generic", "screw"])
def test_query_at_baseline_windows(cfg, kind):
    n, domain, w = CONFIGS[cfg]
    rng = np.random.default_rng(sum(map(ord, cfg + kind)))
    C1, C2 = lean_window(rng, w), lean_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    h, origin, c, dom, dcell = grid_consts(n, domain)
    poses = poses_for(kind, rng, 3 if cfg == "C2" else 5, domain, c)
    with ThreadPoolExecutor(max_workers=len(poses)) as pool:
        wants = list(pool.map(lambda p: reference_cascade(C1, C2, False, dom, dcell, p[0], p[1], c), poses))
        l1s = list(pool.map(lambda p: oracle.cascade_term_scales(C1, C2, False, dom, dcell, p[0], p[1], c), poses))
    got32 = [be.cascade(W1, W2, False, dom, dcell, R, t, c, precision="fp32") for R, t in poses]
    got64 = [be.cascade(W1, W2, False, dom, dcell, R, t, c, precision="fp64") for R, t in poses]
    with be.HapticServer(W1, W2, False, dom, dcell, c, precision="fp32"):
        srv32 = [be.cascade(W1, W2, False, dom, dcell, R, t, c, precision="fp32") for R, t in poses]
    for g32, g64, s32, want, l1 in zip(got32, got64, srv32, wants, l1s):
        assert np.all(parity_tol(g32, want, l1, 1e-4)), np.max(np.abs(g32 - want) / np.maximum(np.abs(want), l1))
        assert np.all(parity_tol(g64, want, l1, 1e-10)), np.max(np.abs(g64 - want) / np.maximum(np.abs(want), l1))
        # the session path: same tolerance (its grid may fall back to one-CTA
        # clusters at w = 128, a different association of the CTA partials)
        assert np.all(parity_tol(s32, want, l1, 1e-4))
        scale = np.max(np.abs(want))
        assert np.max(np.abs(g64 - want)) <= 1e-9 * scale
        assert np.max(np.abs(g32 - want)) <= 1e-3 * scale


def test_sweep_C3_cmd_bench_poses():
    import torch

    n, domain, w = CONFIGS["C3"]
    rng = np.random.default_rng(33)
    C1, C2 = lean_window(rng, w), lean_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    h, origin, c, dom, dcell = grid_consts(n, domain)
    Rs, ts = oracle.bench_poses(512, 0.25 * domain, seed=0)
    t_eff = ts - c + np.einsum("nij,j->ni", Rs, c)
    poses = torch.from_numpy(be.pack_poses(Rs, t_eff)).cuda()
    out = be.cascade_batch(W1, W2, False, dom, dcell, c, poses, precision="fp32").cpu().numpy().view(np.complex128)
    idx = [0, 1, 97, 255, 511]
    with ThreadPoolExecutor(max_workers=len(idx)) as pool:
        wants = list(pool.map(lambda i: reference_cascade(C1, C2, False, dom, dcell, Rs[i], t_eff[i], c), idx))
        l1s = list(pool.map(lambda i: oracle.cascade_term_scales(C1, C2, False, dom, dcell, Rs[i], t_eff[i], c), idx))
    for i, want, l1 in zip(idx, wants, l1s):
        assert np.all(parity_tol(out[i], want, l1, 1e-4))


def test_headline_C2_real_assets_through_evaluate():
    """The headline configuration on its stated inputs: GPU-built assets of
    the low-clearance peg-in-hole at 128^3, K=32, queried through the public
    evaluate() along a jittered insertion path, against the reference kernel
    on the very windows the engine uses."""
    sc = scenes.get_scene("peg_in_hole_lowclear")
    m = 64 ** 3
    a1, a2 = sc.build_assets(128, m_prime=m)
    (w1, wrap1), (w2, _) = a1.window(m), a2.window(m)
    C1, C2 = np.asarray(w1), np.asarray(w2)
    g = a1.grid
    c, dom, dcell = g.center(), g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
    rng = np.random.default_rng(20260814)
    cfgs = []
    for z in (0.4, 0.25, 0.1, 0.02, 0.0):
        j = np.deg2rad(0.5) * rng.normal(size=3)
        R = oracle.axis_rotation(3, 0, j[0]) @ oracle.axis_rotation(3, 1, j[1]) @ oracle.axis_rotation(3, 2, j[2])
        cfgs.append(Configuration(R, np.array([0.0, 0.0, z]) + (g.spacing / 4) * rng.normal(size=3)))
    for prec, tol in (("fp32", 1e-4), ("fp64", 1e-10)):
        be.set_precision(prec)
        try:
            evs = [evaluate(a1, a2, cfg, m) for cfg in cfgs]
        finally:
            be.set_precision("fp32")
        for cfg, ev in zip(cfgs, evs):
            R, t = cfg.rotation, cfg.translation
            te = t - c + R @ c
            ref = reference_cascade(C1, C2, wrap1, dom, dcell, R, te, c)
            l1 = oracle.cascade_term_scales(C1, C2, wrap1, dom, dcell, R, te, c)
            got = np.concatenate([[-ev.energy], ev.force, ev.torque])
            want = np.concatenate([[ref[0].real], ref[1:4].real, ref[4:7].real])
            assert np.all(np.abs(got - want) <= tol * np.maximum(np.abs(want), l1.real)), (prec, got, want)


class _Pair:
    """Minimal asset pair for score_field_device (windows already centred)."""

    def __init__(self, grid, win, wrap):
        self.grid, self._w = grid, (win, wrap)

    def window(self, m_prime=None):
        return self._w


@pytest.fixture(scope="module")
def land256():
    n, h = 256, 5.42 / 256
    origin = -0.5 * 5.42
    rng = np.random.default_rng(256)
    C1, C2 = lean_window(rng, n), lean_window(rng, n)
    R = oracle.bench_poses(1, 1.0, seed=1)[0][0]
    want = oracle.score_field(C1, C2, True, (n,) * 3, (origin,) * 3, h, R).ravel()
    l1 = oracle.score_field_scale(C1, C2, True, (n,) * 3, h, R)
    g = SampleGrid(3, (n,) * 3, (origin,) * 3, h)
    return g, C1, C2, R, want, l1


@pytest.mark.parametrize("prec,tol", [(32, 1e-4), (64, 1e-9)])
def test_landscape_256_full_spectrum(land256, prec, tol):
    g, C1, C2, R, want, l1 = land256
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    land = score_field_device(_Pair(g, W1, True), _Pair(g, W2, True), R, None, precision=prec)
    got = land.cpu().numpy().astype(np.complex128)
    err = np.abs(got - want)
    assert np.all(err <= tol * np.maximum(np.abs(want), l1)), float(np.max(err / np.maximum(np.abs(want), l1)))
    if prec == 64:
        assert np.max(err) <= 1e-9 * np.max(np.abs(want))


@pytest.mark.parametrize("w", [128, 512])
def test_landscape_512_sampled_voxels(w):
    """512^3 landscape; voxel j against the C restatement of the cascade at
    t = p_j (energy.py:309-344 is score_at over the node translations)."""
    n, h = 512, 5.42 / 512
    origin = -0.5 * 5.42
    rng = np.random.default_rng(512 + w)
    C1, C2 = lean_window(rng, w), lean_window(rng, w)
    wrap = w == n
    R = oracle.bench_poses(1, 1.0, seed=1)[0][0]
    g = SampleGrid(3, (n,) * 3, (origin,) * 3, h)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    land = score_field_device(_Pair(g, W1, wrap), _Pair(g, W2, wrap), R, None, precision=32)
    c = g.center()
    dom, dcell = g.delta_omega(), 1.0 / (g.node_count * g.cell_volume)
    # full spectrum: 134M modes per voxel in the C restatement (~30 s each), two voxels
    picks = [(0, 0, 0), (17, 300, 511)]
    if w < n:
        picks += [(n // 2, n // 2, n // 2), (511, 5, 260)] + [tuple(int(v) for v in rng.integers(0, n, 3))
                                                              for _ in range(8)]
    vals = land.reshape(n, n, n)
    got = np.array([complex(vals[p].item()) for p in picks])
    del land, vals
    p_phys = [np.asarray(origin) + h * np.asarray(p, dtype=np.float64) for p in picks]
    with ThreadPoolExecutor(max_workers=len(picks)) as pool:
        wants = list(pool.map(lambda p: oracle.cascade(C1, C2, wrap, dom, dcell, R, p - c + R @ c, c)[0], p_phys))
    # L1 floor from every 4th mode per axis (x 64); 0.9 x keeps the bound on the strict side
    l1 = 0.9 * oracle.score_field_scale(C1, C2, wrap, (n,) * 3, h, R, stride=4 if w == n else 1)
    wants = np.asarray(wants)
    assert np.all(np.abs(got - wants) <= 1e-4 * np.maximum(np.abs(wants), l1)), np.max(np.abs(got - wants) / l1)


@pytest.mark.parametrize("scene,n,which", [("peg_in_hole", 64, "fixed"), ("peg_in_hole", 64, "moving"),
                                           ("gear_pair", 32, "fixed"), ("gear_pair", 32, "moving"),
                                           ("bolt_nut", 32, "fixed"), ("bolt_nut", 32, "moving")])
def test_affinity_at_baseline_geometry(scene, n, which):
    sc = scenes.get_scene(scene)
    g = sc.grid(n)
    solid = getattr(sc, which)
    f = affinity_field(solid, g, sc.kernel)
    want, flags, stats, _, _ = oracle.affinity_values(*solid.element_arrays(), g.dims, g.origin, g.spacing,
                                                      sigma=sc.kernel.sigma, lambda_in=sc.kernel.lambda_in,
                                                      lambda_out=sc.kernel.lambda_out)
    assert f.flags == flags
    for k in ("excluded", "eta_clamped", "worst_residual", "unresolved_nodes", "inside_nodes"):
        assert f.stats[k] == stats[k], k
    np.testing.assert_allclose(f.values, want, rtol=1e-12, atol=1e-12 * np.max(np.abs(want)))
