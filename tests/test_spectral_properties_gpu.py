"""Stage 2 identities the reference's spectral tests pin
(/root/reference/pkg/tests/test_spectral.py:38-255), checked on the GPU
transforms in 2D and 3D: single-harmonic amplitude, round trip, Parseval,
linearity, Hermitian symmetry of real fields, centred truncation and its
zero-padded inverse, low-pass energy ordering, rotate/reflect identities,
GSPC round trips and truncation idempotence."""

import numpy as np
import pytest

from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid
from paper_1711_05017_b200.spectral import (Spectrum, TruncatedSpectrum, forward_dft, inverse_dft, read_spectrum,
                                            rotate_reflect_spectrum, truncate, write_spectrum, zero_padded)

pytestmark = pytest.mark.gpu


def cell_grid(dims, extent=4.0):
    h = extent / dims[0]
    return SampleGrid(len(dims), tuple(dims), tuple(-extent / 2 + h / 2 for _ in dims), h)


def noise(g, seed, real=False):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(g.node_count)
    if not real:
        v = v + 1j * rng.standard_normal(g.node_count)
    return ComplexField(g, v)


GRIDS = [(16, 16), (8, 8, 8), (32, 16), (16, 8, 32)]


@pytest.mark.parametrize("dims", GRIDS)
def test_lattice_harmonic_is_one_bin(dims):
    g = cell_grid(dims)
    k = np.array([2, -3, 1][: g.dimension])
    w = k * np.asarray(g.delta_omega())
    spec = forward_dft(ComplexField(g, np.exp(2j * np.pi * (g.points() @ w)))).reshaped().copy()
    idx = tuple(n // 2 + kk for n, kk in zip(g.dims, k))
    mass = g.node_count * g.cell_volume
    assert spec[idx] == pytest.approx(mass, rel=1e-12)
    spec[idx] = 0
    assert np.max(np.abs(spec)) < 1e-9 * mass


@pytest.mark.parametrize("dims", GRIDS)
def test_round_trip_and_parseval(dims):
    g = cell_grid(dims)
    for seed in range(4):
        f = noise(g, seed)
        spec = forward_dft(f)
        np.testing.assert_allclose(inverse_dft(spec).values, f.values, rtol=0, atol=1e-12)
        lhs = np.sum(np.abs(f.values) ** 2) * g.cell_volume
        rhs = np.sum(np.abs(spec.amplitudes) ** 2) * np.prod(g.delta_omega())
        assert rhs == pytest.approx(lhs, rel=1e-12)


@pytest.mark.parametrize("dims", GRIDS[:2])
def test_linear(dims):
    g = cell_grid(dims)
    a, b = noise(g, 1), noise(g, 2)
    mix = forward_dft(ComplexField(g, (1.5 - 0.25j) * a.values + 3.0 * b.values)).amplitudes
    want = (1.5 - 0.25j) * forward_dft(a).amplitudes + 3.0 * forward_dft(b).amplitudes
    np.testing.assert_allclose(mix, want, atol=1e-10)


@pytest.mark.parametrize("dims", GRIDS)
def test_real_field_is_hermitian(dims):
    g = cell_grid(dims)
    spec = forward_dft(noise(g, 7, real=True)).reshaped()
    inner = spec[(slice(1, None),) * g.dimension]  # entries whose negation is stored
    flipped = inner[(slice(None, None, -1),) * g.dimension]
    np.testing.assert_allclose(flipped, np.conj(inner), atol=1e-10)


@pytest.mark.parametrize("dims,m_prime", [((16, 16), 36), ((16, 16), 64), ((8, 8, 8), 64), ((16, 16, 16), 216)])
def test_truncation_centred_and_padding_inverts(dims, m_prime):
    g = cell_grid(dims)
    spec = forward_dft(noise(g, 3))
    t = truncate(spec, m_prime)
    side = t.window[0]
    sl = tuple(slice(n // 2 - side // 2, n // 2 + side // 2) for n in g.dims)
    np.testing.assert_array_equal(t.reshaped(), spec.reshaped()[sl])
    z = zero_padded(t).reshaped()
    assert np.count_nonzero(z) == np.count_nonzero(spec.reshaped()[sl])
    np.testing.assert_array_equal(z[sl], spec.reshaped()[sl])
    # idempotent: truncating the padded window again changes nothing
    np.testing.assert_array_equal(zero_padded(truncate(zero_padded(t), m_prime)).amplitudes, z.ravel())
    np.testing.assert_array_equal(zero_padded(truncate(spec, g.node_count)).amplitudes, spec.amplitudes)


def test_truncation_rejects_bad_budgets():
    spec = forward_dft(noise(cell_grid((8, 8)), 0))
    for bad in (9, 100 * 100, 3 * 3):
        with pytest.raises(ValueError):
            truncate(spec, bad)


def test_more_modes_never_lose_energy():
    g = cell_grid((16, 16))
    f = noise(g, 11)
    spec = forward_dft(f)
    errs = [np.linalg.norm(inverse_dft(zero_padded(truncate(spec, m))).values - f.values) for m in (16, 64, 256)]
    assert errs[0] >= errs[1] >= errs[2] and errs[2] < 1e-10


@pytest.mark.parametrize("dims", [(16, 16), (8, 8, 8)])
def test_rotate_reflect_identity_negates_frequency(dims):
    g = cell_grid(dims)
    spec = forward_dft(noise(g, 5, real=True))
    out = rotate_reflect_spectrum(spec, np.eye(g.dimension))
    np.testing.assert_allclose(out.amplitudes, np.conj(spec.amplitudes), atol=1e-9)


def test_rotate_reflect_quarter_turn_is_rotated_field():
    g = cell_grid((16, 16))
    f = noise(g, 9, real=True)
    quarter = np.array([[0.0, -1.0], [1.0, 0.0]])
    out = rotate_reflect_spectrum(forward_dft(f), quarter)
    turned = forward_dft(ComplexField(g, np.rot90(f.values.reshape(g.dims), k=1).ravel()))
    np.testing.assert_allclose(out.amplitudes, np.conj(turned.amplitudes), atol=1e-9)


def test_rotate_reflect_truncated_window():
    g = cell_grid((16, 16))
    t = truncate(forward_dft(noise(g, 4)), 36)
    out = rotate_reflect_spectrum(t, np.eye(2)).reshaped()
    assert np.all(out[0, :] == 0) and np.all(out[:, 0] == 0)  # negated first row/column leave the window
    np.testing.assert_allclose(out[1:, 1:], t.reshaped()[1:, 1:][::-1, ::-1], atol=1e-12)
    c, s = np.cos(0.3), np.sin(0.3)
    gen = rotate_reflect_spectrum(truncate(forward_dft(noise(g, 4)), 64), np.array([[c, -s], [s, c]]))
    assert isinstance(gen, TruncatedSpectrum)
    assert np.all(np.isfinite(gen.amplitudes.view(np.float64)))
    src = truncate(forward_dft(noise(g, 4)), 64)
    assert np.max(np.abs(gen.amplitudes)) <= np.max(np.abs(src.amplitudes)) * (1 + 1e-12)


@pytest.mark.parametrize("dims,m_prime", [((8, 8), None), ((16, 16), 64), ((8, 8, 8), 64)])
def test_gspc_round_trip(tmp_path, dims, m_prime):
    g = cell_grid(dims)
    spec = forward_dft(noise(g, 2))
    s = spec if m_prime is None else truncate(spec, m_prime)
    write_spectrum(s, tmp_path / "s.gspc")
    back = read_spectrum(tmp_path / "s.gspc")
    assert type(back) is (Spectrum if m_prime is None else TruncatedSpectrum) and back.grid == g
    scale = np.max(np.abs(s.amplitudes))
    np.testing.assert_allclose(back.amplitudes, s.amplitudes, atol=2e-6 * scale)
