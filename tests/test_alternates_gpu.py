"""The measured-and-kept alternates stay correct: the u-space tiled cascade
(variant 0, gf_set_cascade_variant) against the default direct gather, and
the fused product + z inverse pass (gf_field_zpass) against the product
kernel followed by the z pass."""

import ctypes

import numpy as np
import pytest

from conftest import random_rotation, synthetic_window
from paper_1711_05017_b200 import _lib, backend

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-10), ("fp32", 2e-4)])
def test_tiled_variant_matches_direct(prec, tol):
    import torch

    rng = np.random.default_rng(8)
    w = 32
    W1, W2 = backend.DeviceWindow(synthetic_window(rng, w)), backend.DeviceWindow(synthetic_window(rng, w))
    n = 12
    Rs = np.stack([random_rotation(rng) for _ in range(n)])
    ts = rng.uniform(-1, 1, (n, 3))
    poses = torch.from_numpy(backend.pack_poses(Rs, ts)).cuda()
    outs = []
    try:
        for variant in (1, 0):
            _lib.check(_lib.LIB.gf_set_cascade_variant(variant))
            out = torch.empty((n, 14), dtype=torch.float64, device="cuda")
            backend.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision=prec)
            outs.append(out.cpu().numpy())
    finally:
        _lib.check(_lib.LIB.gf_set_cascade_variant(1))
    scale = np.max(np.abs(outs[0]), axis=0, keepdims=True)
    np.testing.assert_allclose(outs[1], outs[0], atol=tol * np.max(scale), rtol=0)


@pytest.mark.parametrize("prec,wrap", [(64, False), (32, True)])
def test_fused_zpass_matches_product_then_pass(prec, wrap):
    import torch

    rng = np.random.default_rng(9)
    w, n2 = 32, 64
    W1, W2 = backend.DeviceWindow(synthetic_window(rng, w)), backend.DeviceWindow(synthetic_window(rng, w))
    R = np.ascontiguousarray(random_rotation(rng))
    dom = np.full(3, 0.1)
    s = np.array([0.3, -0.2, 0.1])
    dt = torch.complex128 if prec == 64 else torch.complex64
    st = torch.cuda.current_stream().cuda_stream
    fused = torch.empty((w, w, n2), dtype=dt, device="cuda")
    _lib.check(_lib.LIB.gf_field_zpass(W1.handle, W2.handle, int(wrap), _lib.dptr(dom), n2, _lib.dptr(R), _lib.dptr(s),
                                       prec, 0, -1, ctypes.c_void_p(fused.data_ptr()), ctypes.c_void_p(st)))
    q = torch.empty((w, w, w), dtype=dt, device="cuda")
    _lib.check(_lib.LIB.gf_rotate_product(W1.handle, W2.handle, int(wrap), _lib.dptr(dom), _lib.dptr(R), _lib.dptr(s),
                                          prec, ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(st)))
    ref = torch.empty((w, w, n2), dtype=dt, device="cuda")
    si, so = (ctypes.c_int32 * 3)(w, w, w), (ctypes.c_int32 * 3)(w, w, n2)
    _lib.check(_lib.LIB.gf_fft_pass(prec, ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(ref.data_ptr()), si, so, 2,
                                    n2, 1, 0, 1, 0.0, 0.0, 1.0, ctypes.c_void_p(st)))
    torch.cuda.synchronize()
    a, b = fused.cpu().numpy(), ref.cpu().numpy()
    tol = 1e-12 if prec == 64 else 1e-5
    np.testing.assert_allclose(a, b, atol=tol * np.max(np.abs(b)), rtol=0)
