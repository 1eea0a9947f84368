"""gf_fft_pass (one batched line-FFT pass, fft.cu) against numpy, per code
path: contiguous axis (bulk-copy staged / plain), strided axes (tensor-map
staged, paired-vector, plain), node-ordered and DC-centred (zero-padded /
truncated) lines, the three phase kinds, scale, both precisions."""

import ctypes

import numpy as np
import pytest

from paper_1711_05017_b200 import _lib

pytestmark = pytest.mark.gpu


def numpy_pass(x, axis, n, out_len, in_centered, out_centered, sign, in_phase, out_phase, scale):
    x = np.moveaxis(x, axis, -1)
    Lin = x.shape[-1]
    pos = np.arange(n)
    m_c = np.where(pos < n // 2, pos, pos - n)
    line = np.zeros(x.shape[:-1] + (n,), dtype=np.complex128)
    if in_centered:
        src = m_c + Lin // 2
        ok = (src >= 0) & (src < Lin)
        line[..., pos[ok]] = x[..., src[ok]] * np.exp(2j * np.pi * m_c[ok] * in_phase)
    else:
        line[...] = x * np.exp(2j * np.pi * pos * in_phase)
    y = np.fft.fft(line, axis=-1) if sign < 0 else np.fft.ifft(line, axis=-1) * n
    if out_centered:
        dst = np.arange(out_len)
        p = (dst - out_len // 2) % n
        m = np.where(p < n // 2, p, p - n)
        out = y[..., p] * scale * np.exp(2j * np.pi * m * out_phase)
    else:
        out = y * scale * np.exp(2j * np.pi * pos * out_phase)
    return np.moveaxis(out, -1, axis)


def run_pass(x, axis, n, out_len, in_centered, out_centered, sign, in_phase, out_phase, scale, precision):
    import torch

    dt = torch.complex64 if precision == 32 else torch.complex128
    xin = torch.from_numpy(x).to(dt).cuda()
    oshape = list(x.shape)
    oshape[axis] = out_len
    out = torch.empty(oshape, dtype=dt, device="cuda")
    si = (ctypes.c_int32 * 3)(*x.shape)
    so = (ctypes.c_int32 * 3)(*oshape)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.LIB.gf_fft_pass(precision, ctypes.c_void_p(xin.data_ptr()), ctypes.c_void_p(out.data_ptr()), si,
                                    so, axis, n, int(in_centered), int(out_centered), sign, float(in_phase),
                                    float(out_phase), float(scale), ctypes.c_void_p(st)))
    torch.cuda.synchronize()
    return out.cpu().numpy()


CASES = [
    # n, Lin, Lout, in_centered, out_centered, in_phase, out_phase, scale
    (64, 64, 64, False, False, 0.0, 0.0, 1.0),
    (256, 256, 96, False, True, 0.0, 0.5, 0.25),     # forward window: truncate + (-1)^m
    (512, 512, 128, False, True, 0.0, 0.5, 1.0),
    (512, 200, 512, True, False, 0.5, 0.0, 1.0),     # landscape: zero-pad a centred window
    (128, 128, 128, False, False, 0.1234, -0.377, 2.0),  # general phases
    (512, 512, 512, False, False, 0.0, 0.0, 1.0),
    (32, 32, 20, False, True, 0.0, 0.5, 1.0),
]


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("case", CASES, ids=[f"n{c[0]}_{c[1]}to{c[2]}" for c in CASES])
@pytest.mark.parametrize("s2", [34, 33])
def test_fft_pass_matches_numpy(precision, axis, case, s2):
    n, Lin, Lout, ic, oc, iph, oph, scale = case
    if axis == 2 and s2 == 33:
        pytest.skip("contiguous-axis length is the transform length")
    rng = np.random.default_rng(n + Lin + axis)
    shape = [5, 3, s2]
    shape[axis] = Lin
    x = rng.normal(size=shape) + 1j * rng.normal(size=shape)
    for sign in (-1, 1):
        got = run_pass(x, axis, n, Lout, ic, oc, sign, iph, oph, scale, precision)
        want = numpy_pass(x, axis, n, Lout, ic, oc, sign, iph, oph, scale)
        tol = (2e-5 if precision == 32 else 1e-12) * np.sqrt(n) * np.max(np.abs(x)) * abs(scale)
        np.testing.assert_allclose(got, want, atol=tol, rtol=0)
