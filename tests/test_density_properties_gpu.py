"""Stage 1 properties the reference's descriptor tests pin
(/root/reference/pkg/tests/test_descriptor.py:185-320), on the GPU
pipeline: grid contracts, the inverse-square field is the indicator, stats
and flags, 90-degree rotation equivariance, determinism, indicator area,
vector density, GFLD round trips, and the swept density of a polygonised
disk against an independent angular quadrature (oracle.disk_density)."""

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200.descriptor import (ComplexField, KernelSpec, SampleGrid, affinity_field, indicator_field,
                                              read_field, vector_density, write_field)
from paper_1711_05017_b200.scenes import box_mesh, random_polygon
from paper_1711_05017_b200.solids import Polygon2, Solid

pytestmark = pytest.mark.gpu
SPEC = KernelSpec(sigma=0.5, lambda_in=1.0, lambda_out=3.0)


def square(side):
    h = side / 2
    return Solid(Polygon2([np.array([[-h, -h], [h, -h], [h, h], [-h, h]], float)]))


def cell_grid(n, extent=4.0, d=2):
    h = extent / n
    return SampleGrid(d, (n,) * d, (-extent / 2 + h / 2,) * d, h)


def test_grid_contracts():
    s = square(1.0)
    with pytest.raises(ValueError):
        affinity_field(s, cell_grid(16, d=3), KernelSpec())
    with pytest.raises(ValueError):  # no 2h margin around the square
        affinity_field(s, SampleGrid(2, (8, 8), (-1.0, -1.0), 0.25), KernelSpec())


def test_inverse_square_field_is_the_indicator():
    s = random_polygon(np.random.default_rng(3), n_vertices=8)
    g = cell_grid(32)
    fld = affinity_field(s, g, KernelSpec(family="InverseSquare"))
    ind = indicator_field(s, g)
    keep = np.ones(g.node_count, bool)
    keep[fld.flags] = False
    np.testing.assert_allclose(fld.values[keep], ind.values[keep], atol=1e-9)


def test_stats_flags_and_finiteness():
    fld = affinity_field(square(0.9), cell_grid(32), KernelSpec())
    for key in ("excluded", "eta_clamped", "worst_residual", "inside_nodes", "unresolved_nodes",
                "seconds_distance", "seconds_winding", "seconds_sweep"):
        assert key in fld.stats
    assert fld.stats["seconds_sweep"] > 0 and fld.stats["inside_nodes"] > 0
    assert np.all(np.isfinite(fld.values.view(np.float64)))
    assert fld.flags == sorted(fld.flags)


def test_quarter_turn_equivariance():
    rng = np.random.default_rng(11)
    s = random_polygon(rng, n_vertices=7, r_min=0.4, r_max=0.9)
    R = np.array([[0.0, -1.0], [1.0, 0.0]])
    turned = Solid(Polygon2([np.asarray(s.polygon.loops[0]) @ R.T]))
    g = cell_grid(32)
    f0 = affinity_field(s, g, SPEC).values.reshape(g.dims)
    f1 = affinity_field(turned, g, SPEC).values.reshape(g.dims)
    np.testing.assert_allclose(f1, np.rot90(f0, k=1), rtol=1e-9, atol=1e-12)


def test_repeatable_bit_for_bit():
    g = cell_grid(16)
    a, b = affinity_field(square(0.8), g, KernelSpec()), affinity_field(square(0.8), g, KernelSpec())
    np.testing.assert_array_equal(a.values, b.values)
    assert a.flags == b.flags


def test_indicator_area_and_vector_density():
    g = cell_grid(64)
    ind = indicator_field(square(1.0), g)
    assert ind.values.real.sum() * g.cell_volume == pytest.approx(1.0, rel=0.05)
    g16 = cell_grid(16)
    fld = affinity_field(square(0.8), g16, KernelSpec())
    vec = vector_density(fld)
    P = g16.points()
    for a in range(2):
        np.testing.assert_allclose(vec.components[a].values, fld.values * P[:, a])


def test_gfld_round_trips(tmp_path):
    fld = affinity_field(square(0.9), cell_grid(16), KernelSpec())
    write_field(fld, tmp_path / "f.gfld")
    back = read_field(tmp_path / "f.gfld")
    assert back.grid == fld.grid and back.flags == fld.flags
    np.testing.assert_allclose(back.values, fld.values, rtol=2e-6, atol=1e-7)
    h = 0.5
    g3 = SampleGrid(3, (8, 8, 8), (-2.0 + h / 2,) * 3, h)
    ind = indicator_field(box_mesh((1.0, 1.0, 1.0)), g3)
    write_field(ind, tmp_path / "f3.gfld")
    np.testing.assert_allclose(read_field(tmp_path / "f3.gfld").values, ind.values, atol=1e-7)
    (tmp_path / "junk.gfld").write_bytes(b"NOPE" + b"\x00" * 64)
    with pytest.raises(ValueError):
        read_field(tmp_path / "junk.gfld")
    with pytest.raises(ValueError):
        bad = np.zeros(16, complex)
        bad[3] = np.nan
        ComplexField(cell_grid(4), bad)


def test_swept_disk_matches_angular_quadrature():
    a = 1.0
    th = np.linspace(0, 2 * np.pi, 512, endpoint=False)
    disk = Solid(Polygon2([np.column_stack([a * np.cos(th), a * np.sin(th)])]))
    g = SampleGrid(2, (16, 16), (-2.0 + 0.125, -2.0 + 0.125), 0.25)
    fld = affinity_field(disk, g, SPEC)
    P = g.points()
    r = np.hypot(P[:, 0], P[:, 1])
    keep = np.ones(g.node_count, bool)
    keep[fld.flags] = False
    keep &= np.abs(r - a) > 2.5 * g.spacing  # clear of the rim
    assert keep.sum() > 100
    ref = oracle.disk_density(SPEC.sigma, SPEC.lambda_in, SPEC.lambda_out, a, r[keep])
    np.testing.assert_allclose(fld.values[keep], ref, atol=2e-4 * np.max(np.abs(ref)))
