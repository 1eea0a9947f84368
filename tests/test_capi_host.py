"""CPU-side checks: the C-ABI library loads and exports every declared
symbol; host-side geometry, grids, poses and containers behave like the
reference (no GPU compute here)."""

import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import _lib, backend, scenes, solids
from paper_1711_05017_b200.descriptor import ComplexField, IntegrationPolicy, KernelSpec, SampleGrid, read_field, write_field
from paper_1711_05017_b200.energy import Configuration, _rotated_box, _wrap_mask
from paper_1711_05017_b200.spectral import Spectrum, TruncatedSpectrum, _window_side, read_spectrum, write_spectrum

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "geofield_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(gf_\w+)\s*\(", txt, re.M)))


def test_header_symbols_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 15
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        getattr(lib, s)  # raises AttributeError if not exported
        assert s in _lib.SIGNATURES, f"{s} declared in the header but not bound in _lib"
    for alias, target in _lib.ALIASES.items():
        assert target in syms


def test_session_binding_loads_and_checks_operands():
    # csrc/pyfast.c: the per-frame session query binding shares the ctypes
    # library instance; operands it cannot read in place return None (the
    # caller then takes the ctypes path), engine errors come back as the code
    fast = backend._gf_fast
    assert fast is not None, "_gf_fast extension not built (paper_1711_05017_b200/_build.py build_pyfast)"
    R, t = np.eye(3), np.zeros(3)
    assert fast.server_query(0, R.astype(np.float32), t) is None
    assert fast.server_query(0, R, np.zeros(4)) is None
    assert fast.server_query(0, R.T, t) is None  # not C-contiguous
    assert fast.server_query(0, [[1.0, 0, 0]] * 3, t) is None
    rc = fast.server_query(0, R, t)  # no such server
    assert isinstance(rc, int) and rc == _lib.LIB.gf_server_query(0, R.ravel().ctypes.data_as(_lib.c_dp),
                                                                   t.ctypes.data_as(_lib.c_dp),
                                                                   np.zeros(14).ctypes.data_as(_lib.c_dp))
    assert rc != 0


def test_library_reports_missing_device_loudly():
    if os.environ.get("CUDA_VISIBLE_DEVICES", "") == "" and not _cuda_available():
        rc = _lib.LIB.gf_init(0)
        assert rc != 0
        assert _lib.LIB.gf_last_error()
        with pytest.raises(_lib.EngineError):
            _lib.check(rc)


def _cuda_available():
    import torch

    return torch.cuda.is_available()


def test_backend_switch_matches_reference_errors():
    with pytest.raises(ValueError):
        backend.use("gpu")
    with pytest.raises(RuntimeError):
        backend.use("fallback")
    backend.use("core")
    assert backend.current() == "cuda" and backend.HAVE_CORE


def test_window_side_and_grid():
    assert _window_side(3, 32 ** 3) == 32
    assert _window_side(2, 64) == 8
    with pytest.raises(ValueError):
        _window_side(3, 27)  # odd side
    with pytest.raises(ValueError):
        SampleGrid(3, (12, 16, 16), (0, 0, 0), 0.1)
    g = SampleGrid(3, (16, 16, 16), (-1.0, -1.0, -1.0), 0.125)
    assert g.node_count == 4096
    np.testing.assert_allclose(g.center(), [0.0, 0.0, 0.0])
    np.testing.assert_allclose(g.delta_omega(), [0.5, 0.5, 0.5])
    assert g.node_index((0.01, -0.99, 5.0)) == (8, 0, 15)


def test_configuration_validation():
    with pytest.raises(ValueError):
        Configuration(np.diag([1.0, 1.0, -1.0]), [0, 0, 0])
    cfg = Configuration.from_angle(np.pi / 2, [1.0, 2.0])
    np.testing.assert_allclose(cfg.rotation, [[0, -1], [1, 0]], atol=1e-12)


def test_solid_validation_errors():
    V = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
    F = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]])
    m = solids.TriangleMesh(V, F)
    assert m.genus == 0 and m.signed_volume() > 0
    with pytest.raises(solids.SolidError):
        solids.TriangleMesh(V, F[:3])  # open
    with pytest.raises(solids.SolidError):
        solids.TriangleMesh(V, np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 3, 2]]))  # flipped face
    with pytest.raises(solids.SolidError):
        solids.Polygon2([np.array([[0, 0], [1, 1], [1, 0], [0, 1]], dtype=float)])  # bow tie
    # orientation normalised from inward input
    flipped = solids.TriangleMesh(V, F[:, ::-1])
    assert flipped.signed_volume() > 0


def test_new_generators_are_valid_closed_meshes():
    blk = scenes.bored_block((0.8, 0.8, 0.5), 0.15, 32)
    assert blk.mesh.genus == 1
    peg = scenes.cylinder_peg(0.15, 0.6, 32)
    assert peg.mesh.genus == 0
    np.testing.assert_allclose(peg.measure(), 0.5 * 32 * 0.15 ** 2 * np.sin(2 * np.pi / 32) * 0.6, rtol=1e-12)
    vol = 0.8 * 0.8 * 0.5 - 0.5 * 32 * 0.15 ** 2 * np.sin(2 * np.pi / 32) * 0.5
    np.testing.assert_allclose(blk.measure(), vol, rtol=1e-12)
    nut = scenes.threaded_nut(0.17, 0.2, 0.1, 2, 0.4, 96, 32)
    bolt = scenes.threaded_bolt(0.17, 0.2, 0.1, 2, 96, 32)
    assert nut.mesh.genus == 1 and bolt.mesh.genus == 0
    assert nut.measure() > 0 and bolt.measure() > 0
    g = scenes.gear(24, 0.42, 0.5, 0.3)
    assert g.mesh.genus == 0 and len(g.mesh.faces) == 4 * 24 * 8 - 4


def test_bvh_covers_every_element_once():
    ico = scenes.icosphere(0.5, 2)
    bmin, bmax, left, right, start, count, perm = ico.bvh()
    leaves = left < 0
    assert count[leaves].sum() == len(ico.mesh.faces)
    assert sorted(perm.tolist()) == list(range(len(ico.mesh.faces)))
    assert np.all(count[leaves] <= 4)


def test_containers_round_trip(tmp_path):
    g = SampleGrid(3, (8, 8, 8), (-1.0, -1.0, -1.0), 0.25)
    rng = np.random.default_rng(0)
    vals = rng.normal(size=512) + 1j * rng.normal(size=512)
    f = ComplexField(g, vals, flags=[3, 9])
    write_field(f, tmp_path / "a.gfld")
    back = read_field(tmp_path / "a.gfld")
    np.testing.assert_array_equal(back.values, vals.astype(np.complex64).astype(np.complex128))
    assert back.flags == [3, 9] and back.grid == g
    raw = (tmp_path / "a.gfld").read_bytes()
    assert raw[:4] == b"GFLD" and len(raw) == 56 + 8 * 512 + 4 + 8  # payload at byte 56 in 3D
    s = TruncatedSpectrum(g, 64, vals[:64])
    write_spectrum(s, tmp_path / "b.gspc")
    sb = read_spectrum(tmp_path / "b.gspc")
    assert isinstance(sb, TruncatedSpectrum) and sb.m_prime == 64
    assert (tmp_path / "b.gspc").read_bytes()[:4] == b"GSPC"
    full = Spectrum(g, vals)
    write_spectrum(full, tmp_path / "c.gspc")
    assert isinstance(read_spectrum(tmp_path / "c.gspc"), Spectrum)


def test_wrap_mask_matches_oracle():
    class A:
        pass

    g = SampleGrid(3, (16, 16, 16), (-2.0, -2.0, -2.0), 0.25)
    a1, a2 = A(), A()
    a1.solid_box = (np.array([-0.5, -0.4, -0.3]), np.array([0.5, 0.4, 0.3]))
    a2.solid_box = (np.array([-0.2, -0.2, -0.4]), np.array([0.2, 0.3, 0.4]))
    R = oracle.quat_rotation([0.9, 0.1, -0.3, 0.2])
    got = _wrap_mask(g, a1, a2, R)
    want = oracle.wrap_mask(g.dims, g.origin, g.spacing, a1.solid_box, a2.solid_box, R)
    np.testing.assert_array_equal(got, want)
    lo, hi = _rotated_box(a2.solid_box, np.eye(3))
    np.testing.assert_array_equal(lo, a2.solid_box[0])


def test_bench_pose_generator_is_cmd_bench_order():
    Rs, ts = oracle.bench_poses(5, 1.0, seed=0)
    rng = np.random.default_rng(0)
    q = rng.normal(size=4)
    np.testing.assert_allclose(Rs[0], oracle.quat_rotation(q))
    np.testing.assert_allclose(ts[0], rng.uniform(-1.0, 1.0, 3))


def test_haptic_realtime_enter_leave_restores_thread_state():
    """HapticSession.run's servo-thread setup (pin + SCHED_FIFO) is undone on exit."""
    import os

    from paper_1711_05017_b200 import haptic

    if not hasattr(os, "sched_setaffinity"):
        pytest.skip("no sched_setaffinity")
    aff, pol = os.sched_getaffinity(0), os.sched_getscheduler(0)
    state = haptic._enter_realtime()
    if state[2]:
        assert len(os.sched_getaffinity(0)) == 1 and os.sched_getscheduler(0) == os.SCHED_FIFO
    haptic._leave_realtime(state)
    assert os.sched_getaffinity(0) == aff and os.sched_getscheduler(0) == pol
