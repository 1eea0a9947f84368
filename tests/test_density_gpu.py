"""Stage 1 on the GPU vs the oracle and the reference's golden fields.

Bit-exact: distances, occupancy (winding >= 0.5), excluded/unresolved flags,
residuals and clamp counts.  Values (through exp/atan2): 1e-12 relative.
"""

import os

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import backend, scenes
from paper_1711_05017_b200.descriptor import IntegrationPolicy, KernelSpec, SampleGrid, affinity_field, indicator_field

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_small.npz"))
KERNEL = KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0)


def test_distance_and_winding_bitwise():
    rng = np.random.default_rng(1)
    for solid in (scenes.icosphere(0.4, 2), scenes.bored_block((0.8, 0.8, 0.5), 0.15, 32),
                  scenes.random_polygon(rng, 11)):
        d = solid.dimension
        P = rng.uniform(-0.9, 0.9, size=(2000, d))
        elems = solid.element_arrays()[0]
        np.testing.assert_array_equal(backend.distance_batch(solid, P), oracle.distance(elems, P))
        w_gpu, w_cpu = backend.winding_batch(solid, P), oracle.winding(elems, P)
        np.testing.assert_allclose(w_gpu, w_cpu, rtol=0, atol=1e-12)
        np.testing.assert_array_equal(w_gpu >= 0.5, w_cpu >= 0.5)


def test_distance_culled_on_thread_mesh_bitwise():
    """Large distance batches take the tile-culled kernel (Morton tiles,
    vertex upper bound, running minimum): on the ~10^5-face nut, points on and
    just off the surface and far away give the brute-force minimum exactly."""
    rng = np.random.default_rng(7)
    solid = scenes.get_scene("bolt_nut").fixed
    elems = solid.element_arrays()[0]
    verts = elems.reshape(-1, 3)
    near = verts[rng.integers(0, len(verts), 3000)] + rng.normal(scale=1e-3, size=(3000, 3))
    on = verts[rng.integers(0, len(verts), 500)]  # exactly on the surface: distance 0
    far = rng.uniform(-2.0, 2.0, size=(1500, 3))
    P = np.concatenate([near, on, far])
    np.testing.assert_array_equal(backend.distance_batch(solid, P), oracle.distance(elems, P))


def test_sweep_decisions_bitwise_values_tight():
    rng = np.random.default_rng(2)
    for solid in (scenes.icosphere(0.4, 2), scenes.random_polygon(rng, 9)):
        d = solid.dimension
        P = rng.uniform(-0.8, 0.8, size=(500, d))
        elems, normals, meas = solid.element_arrays()
        xi = np.maximum(oracle.distance(elems, P), 0.01)
        gconst = 1 / (4 * np.pi) if d == 3 else 1 / (2 * np.pi)
        got, gres, gcl = backend.sweep_batch(solid, P, xi, 0.5, gconst, 0.02, 16, 0.01)
        want, wres, wcl = oracle.sweep(elems, normals, meas, P, xi, 0.5, gconst, 0.02, 16, 0.01)
        np.testing.assert_array_equal(gres, wres)
        assert gcl == wcl
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-14 * np.max(np.abs(want)))


@pytest.mark.parametrize("name,key", [("socket", "fixed"), ("peg", "moving")])
def test_affinity_field_matches_reference(name, key):
    peg = scenes.get_scene("peg3d")
    g = peg.grid(16)
    f = affinity_field(getattr(peg, key), g, KERNEL)
    want = GOLD[f"aff3d_{name}_values"]
    np.testing.assert_allclose(f.values, want, rtol=1e-12, atol=1e-12 * np.max(np.abs(want)))
    assert f.flags == GOLD[f"aff3d_{name}_flags"].tolist()
    stats = [f.stats[k] for k in ("excluded", "eta_clamped", "worst_residual", "unresolved_nodes", "inside_nodes")]
    np.testing.assert_array_equal(stats, GOLD[f"aff3d_{name}_stats"])


def test_affinity_field_2d_and_icosphere():
    rng = np.random.default_rng(20260814)
    fixed = scenes.random_polygon(rng, n_vertices=9, r_min=0.45, r_max=0.8)
    moving = scenes.random_polygon(rng, n_vertices=7, r_min=0.3, r_max=0.55)
    g = scenes.grid_for_pair(fixed, moving, 32)
    f = affinity_field(fixed, g, KERNEL)
    np.testing.assert_allclose(f.values, GOLD["aff2d_fixed_values"], rtol=1e-12,
                               atol=1e-12 * np.max(np.abs(GOLD["aff2d_fixed_values"])))
    assert f.flags == GOLD["aff2d_fixed_flags"].tolist()
    ico, box = scenes.icosphere(0.5, 2), scenes.box_mesh((0.8, 1.0, 0.6))
    gi = scenes.grid_for_pair(box, ico, 16)
    fi = affinity_field(ico, gi, KERNEL)
    np.testing.assert_allclose(fi.values, GOLD["aff3d_ico_values"], rtol=1e-12,
                               atol=1e-12 * np.max(np.abs(GOLD["aff3d_ico_values"])))
    assert fi.flags == GOLD["aff3d_ico_flags"].tolist()
    np.testing.assert_array_equal(indicator_field(box, gi).values, GOLD["ind3d_box_values"])


def test_affinity_field_new_geometry_matches_oracle():
    sc = scenes.get_scene("peg_in_hole")
    g = sc.grid(32)
    for solid in (sc.fixed, sc.moving):
        f = affinity_field(solid, g, KERNEL)
        want, flags, stats, _, _ = oracle.affinity_values(*solid.element_arrays(), g.dims, g.origin, g.spacing,
                                                          sigma=0.5, lambda_in=1.0, lambda_out=3.0)
        np.testing.assert_allclose(f.values, want, rtol=1e-12, atol=1e-12 * np.max(np.abs(want)))
        assert f.flags == flags
        for k in ("excluded", "eta_clamped", "worst_residual", "unresolved_nodes", "inside_nodes"):
            assert f.stats[k] == stats[k], k


def test_affinity_deterministic_and_inverse_square():
    ico = scenes.icosphere(0.5, 1)
    g = SampleGrid(3, (16, 16, 16), (-1.0, -1.0, -1.0), 0.125)
    a = affinity_field(ico, g, KERNEL).values
    b = affinity_field(ico, g, KERNEL).values
    np.testing.assert_array_equal(a, b)
    inv = affinity_field(ico, g, KernelSpec(family="InverseSquare"))
    wind = oracle.winding(ico.element_arrays()[0], g.points())
    want = oracle.neighbor_average(wind.astype(np.complex128), oracle.distance(ico.element_arrays()[0],
                                                                               g.points()) < 0.25 * g.spacing, g.dims)
    np.testing.assert_allclose(inv.values, want, atol=1e-12)


@pytest.mark.parametrize("scene,n", [("peg3d", 32), ("peg2d", 64)])
def test_node_slabs_bit_identical_to_whole_grid(scene, n):
    """The multi-GPU node-slab path (gf_affinity_planes with halo planes, one
    call per rank) reassembles to exactly the single-GPU field."""
    import torch

    from paper_1711_05017_b200 import parallel
    from paper_1711_05017_b200.descriptor import _unit_constant

    sc = scenes.get_scene(scene)
    g = sc.grid(n)
    pol = IntegrationPolicy()
    args = (1, KERNEL.sigma, _unit_constant(g.dimension), KERNEL.lambda_in, KERNEL.lambda_out, pol.max_solid_angle,
            pol.max_recursion_depth, pol.eta_floor)
    v0, f0, (c0, w0, _, _) = backend.affinity_grid(sc.fixed, g, *args)
    for world in (2, 3, 5):
        vs, fs, cl, wr = [], [], 0, 0.0
        for p0, k, lo, hi in parallel.density_slab_plan(g.dims[0], world):
            v, f, (c, w, _, _) = backend.affinity_planes(sc.fixed, g, p0, k, lo, hi, *args)
            vs.append(v)
            fs.append(f)
            cl += c
            wr = max(wr, w)
        assert torch.equal(torch.cat(vs), v0) and torch.equal(torch.cat(fs), f0)
        assert cl == c0 and wr == w0
