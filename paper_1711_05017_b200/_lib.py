"""ctypes binding of libgeofield_b200.so (the C ABI in include/geofield_b200.h).

There is no CPU fallback: if the shared library is missing the import fails,
and if no CUDA device is present every compute entry point raises
RuntimeError with the CUDA error text.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgeofield_b200.so")

c_dp = ctypes.POINTER(ctypes.c_double)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_vp = ctypes.c_void_p

# name -> (restype, argtypes); kept in sync with include/geofield_b200.h
SIGNATURES = {
    "gf_init": (ctypes.c_int, [ctypes.c_int]),
    "gf_last_error": (ctypes.c_char_p, []),
    "gf_version": (ctypes.c_int, []),
    "gf_window_create": (ctypes.c_int, [c_dp, ctypes.c_int, c_i32p, c_u64p]),
    "gf_window_create_device": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32p, c_u64p, c_vp]),
    "gf_window_destroy": (ctypes.c_int, [ctypes.c_uint64]),
    "gf_window_device_ptr": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(c_vp)]),
    "gf_cascade": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, ctypes.c_double,
                                  c_dp, c_dp, c_dp, ctypes.c_int, c_dp]),
    # same symbol bound with void* arguments for the per-query fast path
    "gf_cascade_fast": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_vp, ctypes.c_double,
                                       c_vp, c_vp, c_vp, ctypes.c_int, c_vp]),
    "gf_cascade_batch": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, ctypes.c_double,
                                        c_dp, ctypes.c_int, ctypes.c_int64, c_vp, c_vp, c_vp]),
    "gf_cascade_serial": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, ctypes.c_double,
                                         c_dp, ctypes.c_int, ctypes.c_int64, c_vp, c_vp, c_vp]),
    "gf_measure_fma_peak": (ctypes.c_int, [ctypes.c_int, c_dp]),
    "gf_measure_roundtrip": (ctypes.c_int, [ctypes.c_int, c_dp]),
    "gf_measure_launch": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, c_dp, c_dp]),
    "gf_measure_stalls": (ctypes.c_int, [ctypes.c_double, ctypes.c_double, c_dp]),
    "gf_distance_winding": (ctypes.c_int, [ctypes.c_int, c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, c_dp, c_dp]),
    "gf_sweep": (ctypes.c_int, [ctypes.c_int, c_dp, c_dp, c_dp, ctypes.c_int64, c_dp, c_dp, ctypes.c_int64,
                                ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double,
                                c_dp, c_dp, c_i64p]),
    "gf_affinity_grid": (ctypes.c_int, [ctypes.c_int, c_dp, c_dp, c_dp, ctypes.c_int64, c_i32p, c_dp,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_double, c_vp, c_vp, c_dp, c_vp]),
    "gf_winding_grid": (ctypes.c_int, [ctypes.c_int, c_dp, ctypes.c_int64, c_i32p, c_dp, ctypes.c_double, c_vp,
                                       c_vp]),
    "gf_affinity_planes": (ctypes.c_int, [ctypes.c_int, c_dp, c_dp, c_dp, ctypes.c_int64, c_i32p, c_dp,
                                          ctypes.c_double, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                          ctypes.c_double, c_vp, c_vp, c_dp, c_vp]),
    "gf_fft_pass_scatter": (ctypes.c_int, [ctypes.c_int, c_vp, c_i32p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_int, c_i32p, ctypes.POINTER(ctypes.c_uint64),
                                           ctypes.c_int, c_vp]),
    "gf_fft_pass": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_i32p, c_i32p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, c_vp]),
    "gf_rotate_product": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, c_dp, c_dp,
                                         ctypes.c_int, c_vp, c_vp]),
    "gf_rotate_product_planes": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, c_dp, c_dp,
                                                ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, c_vp]),
    "gf_score_field": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, c_i32p, c_dp, c_dp,
                                      ctypes.c_double, ctypes.c_int, c_vp, c_vp, c_vp, c_vp]),
    "gf_set_cascade_debug": (ctypes.c_int, [c_vp]),
    "gf_phase_window": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32p, c_dp, c_dp, c_vp]),
    "gf_wrap_mask": (ctypes.c_int, [c_vp, ctypes.c_int, c_i32p, c_u8p, c_vp]),
    "gf_vector_torque": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                                        c_dp, ctypes.c_double, c_dp, c_dp, c_dp, c_dp]),
    "gf_server_start": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, c_dp, ctypes.c_double, c_dp,
                                       ctypes.c_int, ctypes.c_double, ctypes.c_int, c_u64p]),
    "gf_server_query": (ctypes.c_int, [ctypes.c_uint64, c_dp, c_dp, c_dp]),
    "gf_server_query_fast": (ctypes.c_int, [ctypes.c_uint64, c_vp, c_vp, c_vp]),
    "gf_server_last_timing": (ctypes.c_int, [ctypes.c_uint64, c_dp]),
    "gf_server_stop": (ctypes.c_int, [ctypes.c_uint64]),
    "gf_set_cascade_run_length": (ctypes.c_int, [ctypes.c_int]),
}


# extra Python-side bindings of an exported symbol (name -> symbol)
ALIASES = {"gf_cascade_fast": "gf_cascade", "gf_server_query_fast": "gf_server_query"}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()')"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if name in ALIASES:
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    for alias, target in ALIASES.items():
        fn = ctypes.CFUNCTYPE(SIGNATURES[alias][0], *SIGNATURES[alias][1])((target, lib))
        setattr(lib, alias, fn)
    return lib


LIB = _load()


ESTOPPED = -4  # gf status: the haptic server has stopped (idle timeout); fall back to a launch


class EngineError(RuntimeError):
    """A C-ABI call failed (CUDA error or invalid argument at the boundary)."""


def check(rc):
    if rc != 0:
        msg = LIB.gf_last_error()
        raise EngineError(f"geofield_b200 error {rc}: {msg.decode() if msg else 'unknown'}")


_initialised = set()


def ensure_device(device=None):
    """Bind the calling thread to a CUDA device (default: torch's current one)."""
    import threading

    if device is None:
        device = _current_device()
    key = (threading.get_ident(), int(device))
    if key not in _initialised:
        check(LIB.gf_init(int(device)))
        _initialised.add(key)
    return int(device)


def _current_device():
    import torch

    return torch.cuda.current_device() if torch.cuda.is_available() else 0


def dptr(a):
    """ctypes double* of a C-contiguous float64/complex128 numpy array."""
    return a.ctypes.data_as(c_dp)
