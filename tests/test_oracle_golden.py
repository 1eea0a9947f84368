"""Pin the CPU oracle (and the host-side geometry mirror) to the reference.

Golden fixtures come from the unmodified reference package
(tests/golden/make_golden.py); oracle/_ref is the reference's own Cython
core compiled from /root/reference (skipped where it was not built).
"""

import os

import numpy as np
import pytest

import oracle
from conftest import lattice_rotations_3d, random_rotation, synthetic_window
from paper_1711_05017_b200 import scenes

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_small.npz"))
KERNEL = dict(sigma=0.5, lambda_in=1.0, lambda_out=3.0)


def grid_of(key):
    n, o, h = GOLD[key]
    return (int(n),) * 3, (o,) * 3, h


def test_geometry_matches_reference():
    peg = scenes.get_scene("peg3d")
    np.testing.assert_array_equal(peg.fixed.mesh.triangles, GOLD["geom_socket_tri"])
    np.testing.assert_array_equal(peg.moving.mesh.triangles, GOLD["geom_peg_tri"])
    np.testing.assert_array_equal(scenes.icosphere(0.5, 2).mesh.triangles, GOLD["geom_ico_tri"])
    np.testing.assert_array_equal(scenes.box_mesh((0.8, 1.0, 0.6)).mesh.triangles, GOLD["geom_box_tri"])
    np.testing.assert_array_equal(scenes.lbracket(0.4).mesh.triangles, GOLD["geom_lbracket_tri"])
    rng = np.random.default_rng(20260814)
    poly = scenes.random_polygon(rng, n_vertices=9, r_min=0.45, r_max=0.8)
    np.testing.assert_array_equal(poly.polygon.seg_a, GOLD["geom_poly2_a"])
    np.testing.assert_array_equal(poly.polygon.seg_b, GOLD["geom_poly2_b"])


@pytest.mark.parametrize("name,solid_key", [("socket", "fixed"), ("peg", "moving")])
def test_oracle_affinity_3d_matches_reference(name, solid_key):
    peg = scenes.get_scene("peg3d")
    solid = getattr(peg, solid_key)
    dims, origin, h = grid_of("aff3d_grid")
    values, flags, stats, _, _ = oracle.affinity_values(*solid.element_arrays(), dims, origin, h, **KERNEL)
    want = GOLD[f"aff3d_{name}_values"]
    np.testing.assert_allclose(values, want, rtol=1e-12, atol=1e-12 * np.max(np.abs(want)))
    assert flags == GOLD[f"aff3d_{name}_flags"].tolist()
    got_stats = [stats[k] for k in ("excluded", "eta_clamped", "worst_residual", "unresolved_nodes", "inside_nodes")]
    np.testing.assert_array_equal(got_stats, GOLD[f"aff3d_{name}_stats"])


def test_oracle_affinity_icosphere_and_indicator():
    ico = scenes.icosphere(0.5, 2)
    dims, origin, h = grid_of("aff3d_ico_grid")
    values, flags, _, _, _ = oracle.affinity_values(*ico.element_arrays(), dims, origin, h, **KERNEL)
    np.testing.assert_allclose(values, GOLD["aff3d_ico_values"], rtol=1e-12,
                               atol=1e-12 * np.max(np.abs(GOLD["aff3d_ico_values"])))
    assert flags == GOLD["aff3d_ico_flags"].tolist()
    box = scenes.box_mesh((0.8, 1.0, 0.6))
    wind = oracle.winding(box.element_arrays()[0], oracle.grid_points(dims, origin, h))
    np.testing.assert_array_equal((wind >= 0.5).astype(np.complex128), GOLD["ind3d_box_values"])


def test_oracle_affinity_2d():
    rng = np.random.default_rng(20260814)
    fixed = scenes.random_polygon(rng, n_vertices=9, r_min=0.45, r_max=0.8)
    moving = scenes.random_polygon(rng, n_vertices=7, r_min=0.3, r_max=0.55)
    n, o, h = GOLD["aff2d_grid"]
    dims, origin = (int(n),) * 2, (o,) * 2
    va, fa, _, _, _ = oracle.affinity_values(*fixed.element_arrays(), dims, origin, h, **KERNEL)
    vb, _, _, _, _ = oracle.affinity_values(*moving.element_arrays(), dims, origin, h, **KERNEL)
    np.testing.assert_allclose(va, GOLD["aff2d_fixed_values"], rtol=1e-12,
                               atol=1e-12 * np.max(np.abs(GOLD["aff2d_fixed_values"])))
    assert fa == GOLD["aff2d_fixed_flags"].tolist()
    np.testing.assert_allclose(vb, GOLD["aff2d_moving_values"], rtol=1e-12,
                               atol=1e-12 * np.max(np.abs(GOLD["aff2d_moving_values"])))


def _peg_assets():
    peg = scenes.get_scene("peg3d")
    dims, origin, h = grid_of("aff3d_grid")
    f1 = oracle.affinity_values(*peg.fixed.element_arrays(), dims, origin, h, **KERNEL)[0]
    f2 = oracle.affinity_values(*peg.moving.element_arrays(), dims, origin, h, **KERNEL)[0]
    return peg, dims, origin, h, f1, f2


def test_oracle_spectra_match_reference():
    _, dims, origin, h, f1, _ = _peg_assets()
    A = oracle.forward_dft(f1, dims, origin, h)
    scale = np.max(np.abs(GOLD["spec3d_fixed_full"]))
    np.testing.assert_allclose(A.ravel(), GOLD["spec3d_fixed_full"], atol=1e-12 * scale)
    np.testing.assert_allclose(oracle.center_window(A, dims, origin, h, 8), GOLD["win3d_fixed_m512"],
                               atol=1e-12 * scale)
    np.testing.assert_allclose(oracle.center_window(A, dims, origin, h), GOLD["win3d_fixed_full"], atol=1e-12 * scale)
    # the centred-DFT identity
    C = h ** 3 * np.fft.fftshift(np.fft.fftn(np.fft.ifftshift(f1.reshape(dims))))
    np.testing.assert_allclose(C, GOLD["win3d_fixed_full"], atol=1e-12 * scale)


def test_oracle_evaluate_matches_reference():
    _, dims, origin, h, f1, f2 = _peg_assets()
    A1, A2 = oracle.forward_dft(f1, dims, origin, h), oracle.forward_dft(f2, dims, origin, h)
    c = oracle.grid_center(dims, origin, h)
    dom = (1.0 / (dims[0] * h),) * 3
    dcell = 1.0 / (np.prod(dims) * h ** 3)
    for pose, want in zip(GOLD["eval3d_poses"], GOLD["eval3d_results"]):
        R, t, mp = pose[:9].reshape(3, 3), pose[9:12], int(pose[12])
        w = None if mp in (0, int(np.prod(dims))) else round(mp ** (1 / 3))  # m' = N^d is the full spectrum
        C1 = oracle.center_window(A1, dims, origin, h, w)
        C2 = oracle.center_window(A2, dims, origin, h, w)
        res = oracle.cascade(C1, C2, w is None, dom, dcell, R, t - c + R @ c, c)
        got = np.concatenate([[res[0].real, res[0].imag], res[1:4].real, res[4:7].real])
        np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-9 * np.max(np.abs(want)))


def test_oracle_score_field_matches_reference():
    peg, dims, origin, h, f1, f2 = _peg_assets()
    A1, A2 = oracle.forward_dft(f1, dims, origin, h), oracle.forward_dft(f2, dims, origin, h)
    R = GOLD["field3d_R"]
    for w, key in ((8, "field3d_m512"), (None, "field3d_full")):
        C1 = oracle.center_window(A1, dims, origin, h, w)
        C2 = oracle.center_window(A2, dims, origin, h, w)
        land = oracle.score_field(C1, C2, w is None, dims, origin, h, R)
        want = GOLD[key]
        np.testing.assert_allclose(land.ravel(), want, atol=1e-11 * np.max(np.abs(want)))
    mask = oracle.wrap_mask(dims, origin, h, peg.fixed.bbox, peg.moving.bbox, R)
    np.testing.assert_array_equal(mask.ravel(), GOLD["field3d_wrap_mask"])


# ---------------------------------------------------------------------------
# against the reference's own compiled kernels (oracle/_ref)

CORE = oracle.ref_core()
needs_ref = pytest.mark.skipif(CORE is None, reason="oracle/_ref not built (make -C oracle ref)")


@needs_ref
@pytest.mark.parametrize("w,wrap", [(8, False), (10, True), (16, False)])
def test_oracle_cascade_equals_reference_core(w, wrap):
    rng = np.random.default_rng(w)
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    rots = [random_rotation(rng) for _ in range(3)] + lattice_rotations_3d()[::8]
    for R in rots:
        t, c = rng.normal(size=3), rng.normal(size=3)
        a = oracle.cascade(C1, C2, wrap, (0.1, 0.1, 0.1), 0.3, R, t, c)
        b = CORE.cascade_3d(C1, C2, wrap, 0.1, 0.1, 0.1, 0.3, R, t, c)
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13 * np.max(np.abs(b)))


@needs_ref
def test_oracle_density_kernels_bitwise_equal_reference_core():
    ico = scenes.icosphere(0.4, 2)
    rng = np.random.default_rng(3)
    P = rng.uniform(-0.7, 0.7, size=(300, 3))
    tri = np.ascontiguousarray(ico.mesh.triangles)
    bvh = ico.bvh()
    want = np.empty(len(P))
    CORE.distance_3d(*bvh, tri, P, want, 0, len(P))
    np.testing.assert_array_equal(oracle.distance(ico.element_arrays()[0], P), want)
    np.testing.assert_array_equal(oracle.distance_bvh(bvh, ico.element_arrays()[0], P), want)
    wref = np.empty(len(P))
    CORE.winding_3d(tri, P, wref, 0, len(P))
    np.testing.assert_array_equal(oracle.winding(ico.element_arrays()[0], P), wref)
    xi = np.maximum(want, 0.01)
    out = np.empty(len(P), dtype=np.complex128)
    resid = np.zeros(len(P))
    clamps = np.zeros(len(P), dtype=np.int64)
    m = ico.mesh
    CORE.sweep_3d(tri, m.normals, m.areas, P, xi, 0.5, 1 / (4 * np.pi), 0.02, 16, 0.01, out, resid, clamps, 0, len(P))
    got, gres, gcl = oracle.sweep(*ico.element_arrays(), P, xi, 0.5, 1 / (4 * np.pi), 0.02, 16, 0.01)
    np.testing.assert_array_equal(got, out)
    np.testing.assert_array_equal(gres, resid)
    assert gcl == int(clamps.sum())
