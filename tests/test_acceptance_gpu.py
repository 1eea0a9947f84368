"""The reference's release-gate criteria that concern the hot path
(/root/reference/pkg/tests/test_acceptance.py:87-392), restated against the
GPU engine in float64 with independent references under oracle/:

1. cascade == real-space brute sum (7 part pairs x 100 lattice configs, 1e-9);
2. winding membership == ray-crossing parity (10^4 off-boundary points/solid);
3. analytic force/torque == central differences on the 256^2 demo scene;
4. indicator scores == overlap measure within one cell volume;
7. the full-spectrum landscape's well sits at the snap translation (512^2);
9. transform identities: round trip, Parseval, direct DFT, engine vs resum."""

import time

import numpy as np
import pytest

import oracle
from conftest import SEED, lattice_rotations_3d
from paper_1711_05017_b200 import backend
from paper_1711_05017_b200.descriptor import ComplexField, IntegrationPolicy, SampleGrid, indicator_field, point_membership
from paper_1711_05017_b200.energy import (Configuration, PartAsset, _rotated_box, rotational_gradient, score_at,
                                          score_field, translational_gradient)
from paper_1711_05017_b200.scenes import box_mesh, get_scene, grid_for_pair, icosphere, lbracket, random_polygon
from paper_1711_05017_b200.spectral import forward_dft, inverse_dft

pytestmark = pytest.mark.gpu
QUARTERS = [np.round(oracle.axis_rotation(2, 0, k * np.pi / 2)) for k in range(4)]


@pytest.fixture(autouse=True)
def fp64_engine():
    prev = backend.precision()
    backend.set_precision("fp64")
    yield
    backend.set_precision(prev)


def pair_assets(fixed, moving, g):
    i1, i2 = indicator_field(fixed, g), indicator_field(moving, g)
    return (i1, i2), (PartAsset.from_field("fixed", i1, solid_box=fixed.bbox),
                      PartAsset.from_field("moving", i2, movable=True, solid_box=moving.bbox))


def seam_free(g, a1, a2, R, n, rng):
    glo, ghi = g.box()
    rlo, rhi = _rotated_box(a2.solid_box, R)
    r1 = 0.5 * float(np.linalg.norm(a1.solid_box[1] - a1.solid_box[0]))
    klo = np.ceil((glo + r1 - rlo) / g.spacing).astype(int)
    khi = np.floor((ghi - r1 - rhi) / g.spacing).astype(int)
    return np.stack([rng.integers(klo[a], khi[a] + 1, size=n) for a in range(g.dimension)], axis=1) * g.spacing


def brute(i1, i2, R, t, wrap=False):
    g = i1.grid
    return oracle.brute_score(i1.values, i2.values, g.dims, g.origin, g.spacing, R, t, wrap)


def test_criterion_1_cascade_equals_real_space_sum():
    rng = np.random.default_rng(SEED + 1)
    pairs = [(random_polygon(rng, n_vertices=int(rng.integers(6, 11)), r_min=0.45, r_max=0.85),
              random_polygon(rng, n_vertices=int(rng.integers(5, 9)), r_min=0.3, r_max=0.6)) for _ in range(5)]
    pairs += [(box_mesh((1.0, 1.2, 0.8)), icosphere(0.5)), (lbracket(0.4), box_mesh((0.5, 0.4, 0.3)))]
    t0 = time.perf_counter()
    worst = 0.0
    for fixed, moving in pairs:
        g = grid_for_pair(fixed, moving, 32)
        (i1, i2), (a1, a2) = pair_assets(fixed, moving, g)
        rots = QUARTERS if g.dimension == 2 else lattice_rotations_3d()
        n, err, scale = 0, 0.0, 0.0
        while n < 100:
            R = rots[rng.integers(len(rots))]
            for t in seam_free(g, a1, a2, R, 10, rng):
                s, b = score_at(a1, a2, Configuration(R, t)), brute(i1, i2, R, t)
                err, scale, n = max(err, abs(s - b)), max(scale, abs(b)), n + 1
        worst = max(worst, err / scale)
    assert worst <= 1e-9, worst
    assert time.perf_counter() - t0 < 120.0


def test_criterion_2_winding_membership_equals_ray_parity():
    rng = np.random.default_rng(SEED + 2)
    policy = IntegrationPolicy(max_recursion_depth=24)
    for solid in (box_mesh((1.0, 1.0, 1.0)), icosphere(0.5), lbracket(0.4)):
        lo, hi = solid.bbox
        span, diag = hi - lo, float(np.linalg.norm(hi - lo))
        pts = []
        while len(pts) < 10_000:
            P = lo - 0.1 * span + rng.uniform(size=(12_000, 3)) * 1.2 * span
            pts.extend(P[backend.distance_batch(solid, P) >= 1e-6 * diag].tolist())
        P = np.asarray(pts[:10_000])
        w = point_membership(solid, P, policy)
        inside = oracle.raycast_inside(solid.element_arrays()[0], P, seed=SEED)
        assert np.array_equal(w > 0.5, inside)
        assert np.abs(w[inside] - 1.0).max() <= 0.05 and np.abs(w[~inside]).max() <= 0.05


def test_criterion_3_gradients_equal_central_differences():
    a1, a2 = get_scene("peg2d").build_assets(256)
    rng = np.random.default_rng(SEED + 3)

    def scorer(R, t):
        return score_at(a1, a2, Configuration(R, t))

    wt = wr = 0.0
    t0 = time.perf_counter()
    for _ in range(50):
        cfg = Configuration.from_angle(rng.uniform(0, 2 * np.pi), rng.uniform(-0.8, 0.8, 2))
        tg, rg = translational_gradient(a1, a2, cfg), rotational_gradient(a1, a2, cfg)
        fdt, fdr = oracle.fd_gradient(scorer, cfg.rotation, cfg.translation)
        wt = max(wt, np.linalg.norm(tg - fdt) / np.linalg.norm(fdt))
        wr = max(wr, abs(rg[0] - fdr[0]) / abs(fdr[0]))
    assert wt <= 1e-4 and wr <= 1e-3, (wt, wr)
    assert time.perf_counter() - t0 < 60.0


def test_criterion_4_indicator_score_is_overlap_measure():
    rng = np.random.default_rng(SEED + 4)
    fixed = random_polygon(rng, n_vertices=8, r_min=0.45, r_max=0.85)
    moving = random_polygon(rng, n_vertices=6, r_min=0.3, r_max=0.6)
    g = grid_for_pair(fixed, moving, 32)
    (i1, i2), (a1, a2) = pair_assets(fixed, moving, g)
    dV = g.cell_volume

    def gap(a, b, i, j, R, ts):
        return max(abs(score_at(a, b, Configuration(R, t)).real - brute(i, j, R, t).real) for t in ts)

    assert max(gap(a1, a2, i1, i2, R, seam_free(g, a1, a2, R, 8, rng)) for R in QUARTERS) <= 1e-10
    ts = np.concatenate([seam_free(g, a1, a2, np.eye(2), 10, rng), rng.uniform(-0.5, 0.5, (10, 2)) * g.spacing])
    assert gap(a1, a2, i1, i2, np.eye(2), ts) <= dV
    for _ in range(10):
        R = oracle.axis_rotation(2, 0, rng.uniform(0, 2 * np.pi))
        assert gap(a1, a2, i1, i2, R, seam_free(g, a1, a2, R, 3, rng)) <= dV
    bf, bm = box_mesh((1.0, 0.8, 0.9)), box_mesh((0.5, 0.45, 0.4))
    g3 = grid_for_pair(bf, bm, 16)
    (j1, j2), (b1, b2) = pair_assets(bf, bm, g3)
    rots = lattice_rotations_3d()
    for k in range(6):
        R = rots[rng.integers(len(rots))]
        T = seam_free(g3, b1, b2, R, 4, rng)
        if k % 2:
            T = T + rng.uniform(-0.5, 0.5, T.shape) * g3.spacing
        assert gap(b1, b2, j1, j2, R, T) <= g3.cell_volume


def test_criterion_7_snap_well_is_the_global_minimum():
    sc = get_scene("peg2d")
    a1, a2 = sc.build_assets(512)
    g = a1.grid
    land = score_field(a1, a2, np.eye(2))
    re = np.where(land.wrap_mask.reshape(g.dims), -np.inf, np.real(land.values).reshape(g.dims))
    cell = np.unravel_index(np.argmax(re), g.dims)
    snap = g.node_index(sc.snap_translation)
    assert max(abs(cell[0] - snap[0]), abs(cell[1] - snap[1])) <= 1, (cell, snap)


def test_criterion_9_transform_identities():
    rng = np.random.default_rng(SEED + 9)
    g = SampleGrid(2, (16, 16), (-1.0, -1.0), 0.125)
    v1 = rng.normal(size=256) + 1j * rng.normal(size=256)
    v2 = rng.normal(size=256) + 1j * rng.normal(size=256)
    f1, f2 = ComplexField(g, v1), ComplexField(g, v2)
    spec = forward_dft(f1)
    assert np.abs(inverse_dft(spec).values - v1).max() <= 1e-12
    lhs = np.sum(np.abs(v1) ** 2) * g.cell_volume
    assert abs(lhs - np.sum(np.abs(spec.amplitudes) ** 2) * np.prod(g.delta_omega())) / lhs <= 1e-9
    W = oracle.window_freqs(g.dims, np.asarray(g.delta_omega()))
    direct = oracle.direct_amplitudes(v1, g.dims, g.origin, g.spacing, W)
    assert np.abs(direct - spec.amplitudes).max() / np.abs(spec.amplitudes).max() <= 1e-10
    a1, a2 = PartAsset.from_field("fixed", f1), PartAsset.from_field("moving", f2, movable=True)
    for R in QUARTERS:
        t = rng.uniform(-0.4, 0.4, 2)
        s = score_at(a1, a2, Configuration(R, t))
        c = oracle.cascade_direct(v1, v2, g.dims, g.origin, g.spacing, R, t)
        assert abs(s - c) / abs(c) <= 1e-10
