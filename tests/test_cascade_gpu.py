"""Q1 cascade kernel vs the oracle (C restatement of _core.cascade_3d/2d).

Tolerances (stated): fp32 engine |new - ref| <= 1e-4 * max(|ref|, L1) with
L1 = dcell * sum|summand| per output; fp64 engine
<= 1e-10 relative to max(|ref|, L1) (the reference's own test_backend
cascade tolerance, test_backend.py:79-108).
"""

import numpy as np
import pytest

import oracle
from conftest import lattice_rotations_3d, parity_tol, random_rotation, synthetic_window

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def be():
    from paper_1711_05017_b200 import backend

    return backend


CASES = [(8, False), (16, False), (16, True), (32, False), (12, False), (10, True)]


@pytest.mark.parametrize("w,wrap", CASES)
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_cascade_3d_generic_rotations(be, w, wrap, prec, tol):
    rng = np.random.default_rng(1000 + w + 7 * wrap)
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom = (0.11, 0.11, 0.11)
    dcell = 0.37
    center = rng.normal(size=3)
    for _ in range(4):
        R = random_rotation(rng)
        t = rng.uniform(-3, 3, size=3)
        got = be.cascade(W1, W2, wrap, dom, dcell, R, t, center, precision=prec)
        want = oracle.cascade(C1, C2, wrap, dom, dcell, R, t, center)
        l1 = oracle.cascade_term_scales(C1, C2, wrap, dom, dcell, R, t, center)
        assert np.all(parity_tol(got, want, l1, tol)), (got, want, l1)


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_cascade_3d_lattice_rotations_torque_exact_cell(be, prec, tol):
    """At lattice rotations the float64 floor decision must match the
    reference so the torque takes the same trilinear cell."""
    rng = np.random.default_rng(7)
    w = 16
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom = (1.0 / (16 * 0.3),) * 3  # non-dyadic spacing: ties land on both sides
    for R in lattice_rotations_3d()[::3]:
        t = rng.uniform(-1, 1, size=3)
        got = be.cascade(W1, W2, False, dom, 0.5, R, t, np.array([0.1, -0.2, 0.3]), precision=prec)
        want = oracle.cascade(C1, C2, False, dom, 0.5, R, t, np.array([0.1, -0.2, 0.3]))
        l1 = oracle.cascade_term_scales(C1, C2, False, dom, 0.5, R, t, np.array([0.1, -0.2, 0.3]))
        assert np.all(parity_tol(got, want, l1, tol))


def test_cascade_2d(be):
    rng = np.random.default_rng(3)
    for w, wrap in [(16, False), (32, True)]:
        C1 = synthetic_window(rng, w, 2)
        C2 = synthetic_window(rng, w, 2)
        th = 0.37
        R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        t = np.array([0.3, -0.7])
        c = np.array([0.2, 0.1])
        for prec, tol in [("fp32", 1e-4), ("fp64", 1e-10)]:
            got = be.cascade(C1, C2, wrap, (0.2, 0.2), 0.3, R, t, c, precision=prec)
            want = oracle.cascade(C1, C2, wrap, (0.2, 0.2), 0.3, R, t, c)
            l1 = oracle.cascade_term_scales(C1, C2, wrap, (0.2, 0.2), 0.3, R, t, c)
            assert got.shape == (4,)
            assert np.all(parity_tol(got, want, l1, tol)), (prec, got, want)


def test_cascade_deterministic(be):
    rng = np.random.default_rng(11)
    C1, C2 = synthetic_window(rng, 32), synthetic_window(rng, 32)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    R = random_rotation(rng)
    outs = [be.cascade(W1, W2, False, (0.1,) * 3, 1.0, R, [0.1, 0.2, 0.3], [0, 0, 0]) for _ in range(5)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


def test_cascade_batch_matches_single(be):
    import torch

    rng = np.random.default_rng(5)
    w = 24
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    n = 37
    Rs = np.stack([random_rotation(rng) for _ in range(n)])
    ts = rng.uniform(-2, 2, size=(n, 3))
    poses = torch.from_numpy(be.pack_poses(Rs, ts)).cuda()
    for prec in ("fp32", "fp64"):
        out = be.cascade_batch(W1, W2, False, (0.1,) * 3, 0.5, [0.1, 0.2, 0.3], poses, precision=prec)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.complex128)
        for i in range(0, n, 6):
            want = oracle.cascade(C1, C2, False, (0.1,) * 3, 0.5, Rs[i], ts[i], np.array([0.1, 0.2, 0.3]))
            l1 = oracle.cascade_term_scales(C1, C2, False, (0.1,) * 3, 0.5, Rs[i], ts[i], np.array([0.1, 0.2, 0.3]))
            assert np.all(parity_tol(got[i], want, l1, 1e-4 if prec == "fp32" else 1e-10))


def test_haptic_server_matches_one_shot(be):
    rng = np.random.default_rng(21)
    for w, wrap in ((32, False), (16, True)):
        C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
        W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
        dom, c = (0.11, 0.11, 0.11), np.array([0.1, 0.2, -0.3])
        poses = [(random_rotation(rng), rng.uniform(-1, 1, 3)) for _ in range(20)]
        want = [be.cascade(W1, W2, wrap, dom, 0.4, R, t, c) for R, t in poses]
        with be.HapticServer(W1, W2, wrap, dom, 0.4, c) as srv:
            assert srv.key in be._servers
            got = [be.cascade(W1, W2, wrap, dom, 0.4, R, t, c) for R, t in poses]
        assert srv.key not in be._servers
        for g, w_ in zip(got, want):
            np.testing.assert_array_equal(g, w_)  # same kernel body, same reduction order


def test_session_binding_operand_forms(be):
    """The per-frame session call reads C-contiguous float64 R / t_eff in place
    (csrc/pyfast.c); any other operand form (a transposed view, float32,
    nested lists, a tuple) takes the ctypes path -- same bits either way."""
    assert be._gf_fast is not None
    rng = np.random.default_rng(31)
    w = 32
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, c = (0.09, 0.09, 0.09), (0.1, -0.2, 0.3)
    R = random_rotation(rng)
    t = rng.uniform(-1, 1, 3)
    with be.HapticServer(W1, W2, False, dom, 0.5, c):
        want = be.cascade(W1, W2, False, dom, 0.5, R, t, c)
        forms = [(np.ascontiguousarray(R.T).T, t), (R.tolist(), tuple(t)), (R, list(t))]
        for Rf, tf in forms:
            got = be.cascade(W1, W2, False, dom, 0.5, Rf, tf, c)
            np.testing.assert_array_equal(got, want)
        t32 = t.astype(np.float32)  # float32 operand: the ctypes path widens it exactly
        np.testing.assert_array_equal(be.cascade(W1, W2, False, dom, 0.5, R, t32, c),
                                      be.cascade(W1, W2, False, dom, 0.5, R, t32.astype(np.float64), c))
        assert be.cascade(W1, W2, False, dom, 0.5, R, t, c) is not be.cascade(W1, W2, False, dom, 0.5, R, t, c)


def test_haptic_server_2d_fp64_and_idle_timeout(be):
    import time

    from paper_1711_05017_b200._lib import EngineError

    rng = np.random.default_rng(22)
    # 2D windows, float64 engine: the resident grid answers bit for bit like the launch path
    C1, C2 = synthetic_window(rng, 32, d=2), synthetic_window(rng, 32, d=2)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, c = (0.2, 0.2), np.array([0.1, -0.2])
    poses = []
    for _ in range(10):
        th = rng.uniform(0, 2 * np.pi)
        poses.append((np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]]), rng.uniform(-1, 1, 2)))
    want = [be.cascade(W1, W2, False, dom, 0.3, R, t, c, precision="fp64") for R, t in poses]
    with be.HapticServer(W1, W2, False, dom, 0.3, c, precision="fp64"):
        got = [be.cascade(W1, W2, False, dom, 0.3, R, t, c, precision="fp64") for R, t in poses]
    for g, w_ in zip(got, want):
        assert g.shape == (4,)
        np.testing.assert_array_equal(g, w_)
    # idle timeout: the grid exits by itself; a query then raises, a new session works
    srv = be.HapticServer(W1, W2, False, dom, 0.3, c, precision="fp64", idle_timeout_s=0.05)
    time.sleep(0.3)
    with pytest.raises(EngineError, match="idle timeout"):
        be.check(be.LIB.gf_server_query(srv.id, *[be.dptr(np.ascontiguousarray(x)) for x in
                                                  (np.eye(2), np.zeros(2), np.zeros(14))]))
    # the operator call on that pair is still served: it retires the exited
    # server and falls back to one launch per query (same result)
    assert srv.key in be._servers
    late = be.cascade(W1, W2, False, dom, 0.3, poses[1][0], poses[1][1], c, precision="fp64")
    np.testing.assert_array_equal(late, want[1])
    assert srv.key not in be._servers
    srv.stop()
    with be.HapticServer(W1, W2, False, dom, 0.3, c, precision="fp64"):
        again = be.cascade(W1, W2, False, dom, 0.3, poses[0][0], poses[0][1], c, precision="fp64")
    np.testing.assert_array_equal(again, want[0])


@pytest.mark.parametrize("max_sms", [1, 37, 100])
def test_haptic_server_sm_budget(be, max_sms):
    """A server held to a subset of the SMs answers within the
    parity tolerance of the oracle (its mode split differs from the launch
    path, so not bit for bit), repeatably."""
    rng = np.random.default_rng(23 + max_sms)
    w = 64
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, dcell, c = (0.05,) * 3, 0.3, rng.normal(size=3)
    poses = [(random_rotation(rng), rng.uniform(-1, 1, 3)) for _ in range(3)]
    with be.HapticServer(W1, W2, False, dom, dcell, c, max_sms=max_sms):
        got = [be.cascade(W1, W2, False, dom, dcell, R, t, c) for R, t in poses]
        again = [be.cascade(W1, W2, False, dom, dcell, R, t, c) for R, t in poses]
    for g, a_, (R, t) in zip(got, again, poses):
        np.testing.assert_array_equal(g, a_)
        want = oracle.cascade(C1, C2, False, dom, dcell, R, t, c)
        l1 = oracle.cascade_term_scales(C1, C2, False, dom, dcell, R, t, c)
        assert np.all(parity_tol(g, want, l1, 1e-4))


@pytest.mark.parametrize("w,wrap", [(48, False), (64, True), (96, False)])
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("fp64", 1e-10)])
def test_cascade_3d_long_runs_launch_and_server(be, w, wrap, prec, tol):
    """Windows large enough that every CTA walks several run-axis segments
    (the segment loop's fold and its segment boundaries): launch path vs the
    oracle, and the resident server vs the launch path.  The server grid has
    two CTAs per SM, the launch grid one (cascade.cuh kServerCtasPerSm /
    kLaunchCtasPerSm): the modes are split differently, so the cross-CTA sums
    associate differently -- equal to the last bits of each precision, and
    both within the oracle tolerance above."""
    rng = np.random.default_rng(5000 + w)
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, dcell, c = (0.07, 0.07, 0.07), 0.21, rng.normal(size=3)
    poses = [(random_rotation(rng), rng.uniform(-2, 2, 3)) for _ in range(2)]
    got = [be.cascade(W1, W2, wrap, dom, dcell, R, t, c, precision=prec) for R, t in poses]
    for g, (R, t) in zip(got, poses):
        want = oracle.cascade(C1, C2, wrap, dom, dcell, R, t, c)
        l1 = oracle.cascade_term_scales(C1, C2, wrap, dom, dcell, R, t, c)
        assert np.all(parity_tol(g, want, l1, tol)), (g, want, l1)
    with be.HapticServer(W1, W2, wrap, dom, dcell, c, precision=prec):
        srv = [be.cascade(W1, W2, wrap, dom, dcell, R, t, c, precision=prec) for R, t in poses]
    for s, g, (R, t) in zip(srv, got, poses):
        l1 = oracle.cascade_term_scales(C1, C2, wrap, dom, dcell, R, t, c)
        # per output: a bound on the re-association error of the fixed-order
        # sums, (summation depth ~ 30) x eps x the term scale (L1 of |terms|)
        k = 1e-5 if prec == "fp32" else 1e-13
        assert np.all(np.abs(s - g) <= k * l1), (s, g, l1)


@pytest.mark.parametrize("w,prec", [(64, "fp32"), (32, "fp64"), (96, "fp32")])
def test_serial_loop_matches_single_queries(be, w, prec):
    """gf_cascade_serial (one launch per pose, programmatic dependent launch:
    up to three queries in flight) gives every pose exactly the bits of a lone
    gf_cascade call -- the queries share a 4-slot scratch ring (partials,
    ticket), each slot taken only after its previous user released it."""
    import torch

    rng = np.random.default_rng(70 + w)
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, dcell, c = (0.05,) * 3, 0.3, rng.normal(size=3)
    n = 300
    Rs = np.stack([random_rotation(rng) for _ in range(n)])
    ts = rng.uniform(-1, 1, (n, 3))
    poses = torch.from_numpy(be.pack_poses(Rs, ts)).cuda()
    out = be.cascade_batch(W1, W2, False, dom, dcell, c, poses, precision=prec, serial=True)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.complex128)
    for i in range(n):  # every pose: the 4-slot scratch ring is reused 75 times per slot
        want = be.cascade(W1, W2, False, dom, dcell, Rs[i], ts[i], c, precision=prec)
        np.testing.assert_array_equal(got[i], want)
