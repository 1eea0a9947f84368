"""Query and landscape identities the reference's energy tests pin
(/root/reference/pkg/tests/test_energy.py:33-340), against independent
real-space and direct-sum references restated under oracle/ (numpy):

* exact at lattice rotations and node translations: the cascade equals the
  real-space sum (zero-extended off the seam, circular across it);
* at any real translation the truncated cascade equals the exact
  band-limited mode sum of the low-passed fields;
* generic rotations track the exact sum (interpolation is an approximation);
* gradients match central differences; the landscape matches score_at and
  the circular real-space sum at every node; the wrap mask marks only
  seam-touching translations; indicator scores are overlap areas.

All in the float64 engine (the reference's tolerances)."""

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import backend
from paper_1711_05017_b200.descriptor import ComplexField, KernelSpec, SampleGrid, affinity_field, indicator_field
from paper_1711_05017_b200.energy import (Configuration, PartAsset, _rotated_box, _wrap_mask, evaluate,
                                          rotational_gradient, score_at, score_field, translational_gradient)
from paper_1711_05017_b200.scenes import box_mesh, grid_for_pair, random_polygon
from paper_1711_05017_b200.spectral import forward_dft, inverse_dft, truncate, zero_padded

pytestmark = pytest.mark.gpu
SEED = 20260814
QUARTERS_2D = [np.round(oracle.axis_rotation(2, 0, k * np.pi / 2)) for k in range(4)]


@pytest.fixture(autouse=True)
def fp64_engine():
    prev = backend.precision()
    backend.set_precision("fp64")
    yield
    backend.set_precision(prev)


def fields_of(a):
    g = a.grid
    return dict(dims=g.dims, origin=g.origin, spacing=g.spacing)


@pytest.fixture(scope="module")
def polygons():
    """Two random star polygons on a shared 32^2 grid (skeletal kernel)."""
    rng = np.random.default_rng(SEED)
    fixed = random_polygon(rng, n_vertices=9, r_min=0.45, r_max=0.8)
    moving = random_polygon(rng, n_vertices=7, r_min=0.3, r_max=0.55)
    g = grid_for_pair(fixed, moving, 32)
    k = KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0)
    f1, f2 = affinity_field(fixed, g, k), affinity_field(moving, g, k)
    a1 = PartAsset.from_field("fixed", f1, solid_box=fixed.bbox)
    a2 = PartAsset.from_field("moving", f2, movable=True, solid_box=moving.bbox)
    return dict(fixed=fixed, moving=moving, grid=g, f=(f1, f2), a=(a1, a2))


def indicator_pair(fixed, moving, g):
    i1, i2 = indicator_field(fixed, g), indicator_field(moving, g)
    a1 = PartAsset.from_field("fixed", i1, solid_box=fixed.bbox)
    a2 = PartAsset.from_field("moving", i2, movable=True, solid_box=moving.bbox)
    return (i1, i2), (a1, a2)


def seam_free_node_shifts(g, a1, a2, R, n, rng):
    """Node translations whose moved support stays clear of the wrap seam."""
    glo, ghi = g.box()
    rlo, rhi = _rotated_box(a2.solid_box, R)
    r1 = 0.5 * float(np.linalg.norm(a1.solid_box[1] - a1.solid_box[0]))
    klo = np.ceil((glo + r1 - rlo) / g.spacing).astype(int)
    khi = np.floor((ghi - r1 - rhi) / g.spacing).astype(int)
    assert np.all(khi >= klo)
    return np.stack([rng.integers(klo[a], khi[a] + 1, size=n) for a in range(g.dimension)], axis=1) * g.spacing


def test_exact_vs_real_space_sum_2d(polygons):
    rng = np.random.default_rng(1)
    g = polygons["grid"]
    (i1, i2), (a1, a2) = indicator_pair(polygons["fixed"], polygons["moving"], g)
    for R in QUARTERS_2D:
        for t in seam_free_node_shifts(g, a1, a2, R, 3, rng):
            got = score_at(a1, a2, Configuration(R, t))
            want = oracle.brute_score(i1.values, i2.values, R=R, t=t, wrap=False, **fields_of(a1))
            assert got == pytest.approx(want, rel=1e-10, abs=1e-12)


def test_exact_vs_circular_sum_across_the_seam(polygons):
    g = polygons["grid"]
    a1, a2 = polygons["a"]
    f1, f2 = polygons["f"]
    t = np.array([25 * g.spacing, -13 * g.spacing])
    got = score_at(a1, a2, Configuration(QUARTERS_2D[1], t))
    want = oracle.brute_score(f1.values, f2.values, R=QUARTERS_2D[1], t=t, wrap=True, **fields_of(a1))
    assert got == pytest.approx(want, rel=1e-10, abs=1e-12)


def test_exact_vs_real_space_sum_3d():
    from conftest import lattice_rotations_3d

    rng = np.random.default_rng(2)
    fixed, moving = box_mesh((1.2, 0.8, 0.6)), box_mesh((0.5, 0.5, 0.9))
    g = grid_for_pair(fixed, moving, 16)
    (i1, i2), (a1, a2) = indicator_pair(fixed, moving, g)
    rots = lattice_rotations_3d()
    for R in (rots[0], rots[7], rots[16], rots[23]):
        for t in seam_free_node_shifts(g, a1, a2, R, 2, rng):
            got = score_at(a1, a2, Configuration(R, t))
            want = oracle.brute_score(i1.values, i2.values, R=R, t=t, wrap=False, **fields_of(a1))
            assert got == pytest.approx(want, rel=1e-9, abs=1e-12)


def test_truncated_cascade_is_the_band_limited_sum(polygons):
    """Any real translation, lattice rotations, budgets 16/64/256: the cascade
    over the window equals the exact mode sum of the low-passed fields."""
    rng = np.random.default_rng(3)
    a1, a2 = polygons["a"]
    f1, f2 = polygons["f"]
    for m in (16, 64, 256):
        lp1 = inverse_dft(zero_padded(truncate(forward_dft(f1), m)))
        lp2 = inverse_dft(zero_padded(truncate(forward_dft(f2), m)))
        side = int(round(np.sqrt(m)))
        for R in QUARTERS_2D:
            t = rng.uniform(-0.7, 0.7, size=2)
            got = score_at(a1, a2, Configuration(R, t), m)
            want = oracle.cascade_direct(lp1.values, lp2.values, R=R, t=t, side=side, **fields_of(a1))
            assert got == pytest.approx(want, rel=1e-10, abs=1e-12)


def test_generic_rotation_tracks_the_exact_sum(polygons):
    a1, a2 = polygons["a"]
    f1, f2 = polygons["f"]
    cfg = Configuration.from_angle(0.37, [0.25, -0.1])
    got = score_at(a1, a2, cfg, 64)
    want = oracle.cascade_direct(f1.values, f2.values, R=cfg.rotation, t=cfg.translation, side=8, **fields_of(a1))
    assert got == pytest.approx(want, rel=0.3) and got.real * want.real > 0


def test_full_budget_is_the_default(polygons):
    a1, a2 = polygons["a"]
    cfg = Configuration.from_angle(0.0, [0.3, 0.4])
    assert score_at(a1, a2, cfg) == pytest.approx(score_at(a1, a2, cfg, a1.grid.node_count), rel=1e-12)


def test_gradients_2d_match_central_differences(polygons):
    a1, a2 = polygons["a"]
    cfg = Configuration.from_angle(0.6, [0.2, 0.35])

    def scorer(R, t):
        return score_at(a1, a2, Configuration(R, t), 256)

    fd_t, fd_r = oracle.fd_gradient(scorer, cfg.rotation, cfg.translation)
    np.testing.assert_allclose(translational_gradient(a1, a2, cfg, 256), fd_t, rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(rotational_gradient(a1, a2, cfg, 256), fd_r, rtol=1e-4, atol=1e-9)


def test_vector_path_tracks_central_differences(polygons):
    a1, a2 = polygons["a"]
    cfg = Configuration.from_angle(0.45, [0.3, 0.2])

    def scorer(R, t):
        return score_at(a1, a2, Configuration(R, t))

    vec = rotational_gradient(a1, a2, cfg, path="vector")
    _, fd = oracle.fd_gradient(scorer, cfg.rotation, cfg.translation)
    assert abs(vec[0] - fd[0]) < 0.2 * abs(fd[0]) and vec[0].real * fd[0].real > 0
    with pytest.raises(ValueError):
        rotational_gradient(a1, a2, cfg, path="bogus")


def test_gradients_3d_match_central_differences():
    fixed, moving = box_mesh((1.0, 0.7, 0.5)), box_mesh((0.5, 0.4, 0.8))
    g = grid_for_pair(fixed, moving, 8)
    _, (a1, a2) = indicator_pair(fixed, moving, g)
    R = oracle.axis_rotation(3, 2, 0.4) @ oracle.axis_rotation(3, 0, -0.2)
    cfg = Configuration(R, [0.2, -0.1, 0.15])

    def scorer(Rm, t):
        return score_at(a1, a2, Configuration(Rm, t))

    fd_t, fd_r = oracle.fd_gradient(scorer, R, cfg.translation)
    np.testing.assert_allclose(translational_gradient(a1, a2, cfg), fd_t, rtol=1e-5, atol=1e-8)
    np.testing.assert_allclose(rotational_gradient(a1, a2, cfg), fd_r, rtol=1e-4, atol=1e-8)


def test_evaluate_packaging(polygons):
    a1, a2 = polygons["a"]
    cfg = Configuration.from_angle(0.2, [0.4, 0.1])
    ev = evaluate(a1, a2, cfg, 64)
    assert ev.energy == pytest.approx(-ev.score.real) and ev.modes_used == 64 and ev.eval_time_us > 0
    assert ev.force.shape == (2,) and ev.torque.shape == (1,)
    np.testing.assert_allclose(ev.force, np.real(translational_gradient(a1, a2, cfg, 64)), rtol=1e-12)


def test_landscape_equals_score_at_every_sampled_node(polygons):
    rng = np.random.default_rng(4)
    a1, a2 = polygons["a"]
    g = polygons["grid"]
    R = Configuration.from_angle(0.3, [0, 0]).rotation
    land = score_field(a1, a2, R, 64).values.reshape(g.dims)
    P = g.points().reshape(g.dims + (2,))
    for _ in range(12):
        i, j = rng.integers(0, g.dims[0]), rng.integers(0, g.dims[1])
        assert land[i, j] == pytest.approx(score_at(a1, a2, Configuration(R, P[i, j]), 64), rel=1e-9, abs=1e-12)


def test_full_landscape_equals_circular_sum():
    rng = np.random.default_rng(SEED)
    fixed = random_polygon(rng, n_vertices=8, r_min=0.5, r_max=0.9)
    moving = random_polygon(rng, n_vertices=6, r_min=0.3, r_max=0.6)
    g = grid_for_pair(fixed, moving, 16, center="node")
    k = KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0)
    f1, f2 = affinity_field(fixed, g, k), affinity_field(moving, g, k)
    a1, a2 = PartAsset.from_field("fixed", f1), PartAsset.from_field("moving", f2, movable=True)
    R = QUARTERS_2D[3]
    land = score_field(a1, a2, R).values.reshape(g.dims)
    P = g.points().reshape(g.dims + (2,))
    scale = np.max(np.abs(land))
    for idx in [(0, 0), (3, 14), (8, 8), (15, 1)]:
        want = oracle.brute_score(f1.values, f2.values, R=R, t=P[idx], wrap=True, **fields_of(a1))
        assert land[idx] == pytest.approx(want, abs=1e-11 * scale)


def test_wrap_mask_marks_only_seam_touching(polygons):
    rng = np.random.default_rng(5)
    g = polygons["grid"]
    (i1, i2), (a1, a2) = indicator_pair(polygons["fixed"], polygons["moving"], g)
    R = QUARTERS_2D[1]
    mask = _wrap_mask(g, a1, a2, R)
    assert mask.shape == g.dims and mask.any() and not mask.all()
    P = g.points().reshape(g.dims + (2,))
    clean = np.argwhere(~mask)
    for i, j in clean[rng.integers(0, len(clean), size=10)]:
        a = oracle.brute_score(i1.values, i2.values, R=R, t=P[i, j], wrap=True, **fields_of(a1))
        b = oracle.brute_score(i1.values, i2.values, R=R, t=P[i, j], wrap=False, **fields_of(a1))
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12)
    f1, f2 = polygons["f"]
    bare1, bare2 = PartAsset.from_field("fixed", f1), PartAsset.from_field("moving", f2, movable=True)
    assert not _wrap_mask(g, bare1, bare2, np.eye(2)).any()


def test_landscape_is_deterministic(polygons):
    a1, a2 = polygons["a"]
    R = Configuration.from_angle(1.1, [0, 0]).rotation
    np.testing.assert_array_equal(score_field(a1, a2, R, 64).values, score_field(a1, a2, R, 64).values)


def test_indicator_score_is_the_overlap_area():
    rng = np.random.default_rng(SEED)
    fixed = random_polygon(rng, n_vertices=8, r_min=0.5, r_max=0.9)
    moving = random_polygon(rng, n_vertices=6, r_min=0.3, r_max=0.6)
    g = grid_for_pair(fixed, moving, 64)
    (i1, i2), (a1, a2) = indicator_pair(fixed, moving, g)
    got = score_at(a1, a2, Configuration.from_angle(0.0, [0.0, 0.0]))
    overlap = float(np.sum(i1.values.real.astype(bool) & i2.values.real.astype(bool))) * g.cell_volume
    assert got.imag == pytest.approx(0.0, abs=1e-9)
    assert got.real == pytest.approx(overlap, rel=1e-9, abs=1e-12)


def test_grid_mismatch_and_asset_contracts(polygons):
    a1, _ = polygons["a"]
    f1, f2 = polygons["f"]
    other = SampleGrid(2, (8, 8), (-1.0, -1.0), 0.25)
    stranger = PartAsset.from_field("x", ComplexField(other, np.ones(64, dtype=complex)), movable=True)
    with pytest.raises(ValueError):
        score_at(a1, stranger, Configuration.from_angle(0.0, [0, 0]))
    fixed = PartAsset.from_field("fixed", f1)
    moving = PartAsset.from_field("moving", f2, movable=True)
    assert not fixed.movable and fixed.vector is None and moving.vector is not None
    with pytest.raises(ValueError):
        PartAsset("x", fixed.spectrum, movable=True)
    with pytest.raises(ValueError):
        PartAsset("x", fixed.spectrum, vector=moving.vector, movable=False)
    assert fixed.full_available and fixed.max_modes() == f1.grid.node_count
    lean = PartAsset.from_field("fixed", f1, m_prime=64)
    lean.spectrum = lean.truncated
    assert lean.max_modes() == 64
    lean.window(64)
    lean.window(16)
    for bad in (256, None):
        with pytest.raises(ValueError):
            lean.window(bad)
