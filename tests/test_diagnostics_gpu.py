"""The roofline and platform diagnostics of csrc/diagnostics.cu (bench.py
uses them for the FP32 peak and the C5 platform-stall report)."""

import numpy as np
import pytest

from paper_1711_05017_b200 import _lib

pytestmark = pytest.mark.gpu


def test_fma_peak_is_plausible():
    import ctypes

    _lib.ensure_device(0)
    v = ctypes.c_double()
    _lib.check(_lib.LIB.gf_measure_fma_peak(32, ctypes.byref(v)))
    assert 20.0 < v.value < 200.0  # B200 FP32 FMA pipe: ~72 TFLOP/s


def test_stall_detector_watches_every_sm():
    import torch

    _lib.ensure_device(0)
    out = np.zeros(4)
    _lib.check(_lib.LIB.gf_measure_stalls(0.2, 500.0, _lib.dptr(out)))
    assert int(out[3]) == torch.cuda.get_device_properties(0).multi_processor_count
    assert 0.0 < out[0] < 2e5 and 0 <= out[1] <= out[2]
    bad = np.zeros(4)
    assert _lib.LIB.gf_measure_stalls(0.0, 500.0, _lib.dptr(bad)) != 0  # argument checks
