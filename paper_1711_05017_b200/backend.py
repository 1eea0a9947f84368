"""Operator layer: the reference's `geofield.backend` surface, bound to CUDA.

Mirrors /root/reference/pkg/src/geofield/backend.py (same function names,
argument meaning and error behaviour) but dispatches to the sm_100a kernels
of libgeofield_b200.so through the C ABI (include/geofield_b200.h).  There is
exactly one backend; there is no CPU fallback (`use("fallback")` raises).

Additions over the reference surface:
  * precision control (`set_precision("fp32"|"fp64")`, env
    GEOFIELD_PRECISION): fp32 is the product default (complex64 windows,
    FP32 arithmetic, within 1e-4 of the float64 reference); fp64 reproduces
    the reference's tight tolerances.
  * DeviceWindow: a device-resident window handle; `cascade` accepts these
    (no per-call marshalling) as well as plain numpy windows.
  * cascade_batch: the batched pose sweep (Q3) on device arrays.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _lib
from ._lib import LIB, check, dptr

try:  # CPython binding of the per-frame session query (csrc/pyfast.c); ctypes otherwise
    from . import _gf_fast

    _gf_fast.bind(ctypes.cast(LIB.gf_server_query_fast, ctypes.c_void_p).value)
except ImportError:
    _gf_fast = None

HAVE_CORE = True  # the CUDA engine is the only (and compiled) backend

_NAMES = ("cuda", "core")
_active = "cuda"

_env_prec = os.environ.get("GEOFIELD_PRECISION", "fp32").strip().lower()
if _env_prec not in ("fp32", "fp64"):
    raise ImportError(f"GEOFIELD_PRECISION must be fp32 or fp64, got {_env_prec!r}")
_precision = _env_prec


def current():
    return _active


def use(name):
    """Reference-compatible switch (backend.py:37-44).

    "core"/"cuda" select the compiled CUDA engine; "fallback" is refused
    because this engine deliberately has no CPU path; anything else is a
    ValueError exactly like the reference.
    """
    global _active
    if name == "fallback":
        raise RuntimeError("the B200 engine has no CPU fallback backend")
    if name not in _NAMES:
        raise ValueError(f"unknown backend {name!r}")
    _active = "cuda"


def default_threads():
    """Kept for API compatibility (backend.py:47-52); the GPU ignores it."""
    try:
        n = int(os.environ.get("GEOFIELD_THREADS", "1"))
    except ValueError:
        n = 1
    return max(1, n)


def precision():
    return _precision


def set_precision(name):
    global _precision
    if name not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    _precision = name


def _prec_bits(prec=None):
    return 64 if (prec or _precision) == "fp64" else 32


# ---------------------------------------------------------------------------
# device-resident windows


class DeviceWindow:
    """A centre-referenced window living in HBM behind a C-ABI handle.

    Created from a host complex128 array or a CUDA complex128 torch tensor.
    `np.asarray(win)` materialises the host copy (cached).
    """

    def __init__(self, data, dimension=None):
        _lib.ensure_device()
        self._host = None
        h = ctypes.c_uint64(0)
        if isinstance(data, np.ndarray):
            arr = np.ascontiguousarray(data, dtype=np.complex128)
            d = arr.ndim if dimension is None else dimension
            w = (ctypes.c_int32 * 3)(*(list(arr.shape) + [1] * (3 - arr.ndim)))
            check(LIB.gf_window_create(dptr(arr.view(np.float64)), d, w, ctypes.byref(h)))
            self._host = arr
            self.shape = tuple(arr.shape)
        else:  # torch tensor on the device
            import torch

            t = data.contiguous()
            if t.dtype != torch.complex128:
                t = t.to(torch.complex128)
            d = t.dim() if dimension is None else dimension
            w = (ctypes.c_int32 * 3)(*(list(t.shape) + [1] * (3 - t.dim())))
            st = torch.cuda.current_stream(t.device).cuda_stream
            check(LIB.gf_window_create_device(ctypes.c_void_p(t.data_ptr()), d, w, ctypes.byref(h),
                                              ctypes.c_void_p(st)))
            self._dev = t
            self.shape = tuple(t.shape)
        self.handle = h.value
        self.ndim = len(self.shape)

    def __array__(self, dtype=None, copy=None):
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host if dtype is None else self._host.astype(dtype)

    def ravel(self):
        return np.asarray(self).ravel()

    def reshape(self, *shape):
        return np.asarray(self).reshape(*shape)

    def __getitem__(self, idx):
        return np.asarray(self)[idx]

    def __len__(self):
        return self.shape[0]

    def __del__(self):
        h = getattr(self, "handle", 0)
        if h:
            try:
                LIB.gf_window_destroy(h)
            except Exception:  # interpreter shutdown
                pass


def as_device_window(C):
    return C if isinstance(C, DeviceWindow) else DeviceWindow(np.asarray(C))


# ---------------------------------------------------------------------------
# cascade (Q1) and batched sweep (Q3)


class _QueryBuffers(threading.local):
    """Per-thread pinned-by-address host buffers for the single-query path
    (no per-call array allocation or ctypes pointer construction)."""

    def __init__(self):
        self.arg = np.zeros(24)   # R (9) | t_eff (3) | center (3) | domega (3)
        self.out = np.zeros(14)
        a = self.arg.ctypes.data
        self.pR, self.pt, self.pc, self.pd = (ctypes.c_void_p(a), ctypes.c_void_p(a + 72),
                                              ctypes.c_void_p(a + 96), ctypes.c_void_p(a + 120))
        self.pout = ctypes.c_void_p(self.out.ctypes.data)
        # views used by the session path: one broadcast copy per operand
        self.R33, self.t3 = self.arg[:9].reshape(3, 3), self.arg[9:12]
        self.res3, self.res2 = self.out[:14].view(np.complex128), self.out[:8].view(np.complex128)


_qb = _QueryBuffers()


def _immutable(x):
    return type(x) is tuple or (type(x) is np.ndarray and not x.flags.writeable)


def cascade(C1, C2, wrap, domega, dcell, R, t_eff, center, precision=None):
    """Score + gradients over one retained-mode window (backend.py:153-164).

    Returns complex128[1 + d + n_rot]: [score, dS/dt..., dS/dtheta...], times
    dcell, computed by the CUDA cascade kernel.
    """
    W1 = C1 if type(C1) is DeviceWindow else as_device_window(C1)
    W2 = C2 if type(C2) is DeviceWindow else as_device_window(C2)
    d = W1.ndim
    q = _qb
    bits = 64 if (precision or _precision) == "fp64" else 32
    if _servers and d == 3:
        # session path: only the pose travels (the server holds centre and
        # domega); one C call reads R and t_eff in place (_gf_fast), or two
        # buffer copies and a ctypes call for operands it cannot read
        srv = _servers.get((W1.handle, W2.handle, bool(wrap), bits))
        if srv is not None and srv.dcell == dcell and srv.matches(center, domega):
            r = _gf_fast.server_query(srv.id, R, t_eff) if _gf_fast is not None else None
            if r.__class__ is np.ndarray:
                return r
            if r is None:
                q.R33[...] = R
                q.t3[...] = t_eff
                r = LIB.gf_server_query_fast(srv.id, q.pR, q.pt, q.pout)
                if r == 0:
                    return q.res3.copy()
            if r != _lib.ESTOPPED:
                check(r)
            srv.retire()  # idle-timed out: this and later calls take the launch path
    arg = q.arg
    if d == 3:
        arg[:9] = R.ravel() if type(R) is np.ndarray else np.asarray(R, dtype=np.float64).ravel()
        arg[9:12] = t_eff
        arg[12:15] = center
        arg[15:18] = domega
    else:
        arg[:4] = np.asarray(R, dtype=np.float64).ravel()
        arg[9:11] = t_eff
        arg[12:14] = center
        arg[15:17] = domega
        arg[14] = arg[17] = 0.0
    srv = _servers.get((W1.handle, W2.handle, bool(wrap), bits)) if _servers else None
    rc = _lib.ESTOPPED
    if srv is not None and srv.dcell == dcell and arg[12:18].tobytes() == srv.cd_bytes:
        rc = LIB.gf_server_query_fast(srv.id, q.pR, q.pt, q.pout)
        if rc == _lib.ESTOPPED:
            srv.retire()
    if rc == _lib.ESTOPPED:
        rc = LIB.gf_cascade_fast(W1.handle, W2.handle, 1 if wrap else 0, q.pd, float(dcell), q.pR, q.pt, q.pc, bits,
                                 q.pout)
    if rc:
        check(rc)
    n = 14 if d == 3 else 8
    return q.out[:n].copy().view(np.complex128)


# ---------------------------------------------------------------------------
# persistent haptic server (no kernel launch per query)

_servers = {}


class HapticServer:
    """A resident query grid for one window pair (gf_server_*).

    While it runs, `cascade` calls with the same windows, wrap flag,
    precision and grid constants are answered through its mailbox instead of
    a kernel launch per query.  Use as a context manager (stops on exit); the
    device side also exits on its own after `idle_timeout_s` without queries,
    after which calls fall back to one launch per query.

    `max_sms` > 0 keeps the resident grid on about that many SMs, leaving the
    others free for work issued from other threads while the session runs
    (landscape exports); 0 takes every SM (lowest latency).
    """

    def __init__(self, C1, C2, wrap, domega, dcell, center, precision=None, idle_timeout_s=30.0, max_sms=0):
        self.W1, self.W2 = as_device_window(C1), as_device_window(C2)
        d = self.W1.ndim
        self.bits = 64 if (precision or _precision) == "fp64" else 32
        self.wrap = bool(wrap)
        self.dcell = float(dcell)
        self.dom = np.ascontiguousarray(domega, dtype=np.float64)[:d].copy()
        self.center = np.ascontiguousarray(center, dtype=np.float64)[:d].copy()
        sid = ctypes.c_uint64(0)
        check(LIB.gf_server_start(self.W1.handle, self.W2.handle, int(self.wrap), dptr(self.dom), self.dcell,
                                  dptr(self.center), self.bits, float(idle_timeout_s), int(max_sms),
                                  ctypes.byref(sid)))
        self.id = sid.value
        # one throw-away query: returns once the resident grid is up and its
        # code and windows are warm, so the first real frame pays neither
        R0, z = np.eye(3) if d == 3 else np.eye(2), np.zeros(d)
        warm = np.zeros(14)
        check(LIB.gf_server_query(self.id, dptr(np.ascontiguousarray(R0)), dptr(z), dptr(warm)))
        self.key = (self.W1.handle, self.W2.handle, self.wrap, self.bits)
        cd = np.zeros(6)  # center (3) | domega (3), as laid out in the query buffer
        cd[:d], cd[3:3 + d] = self.center, self.dom
        self.cd_bytes = cd.tobytes()
        self._c_ref = self._d_ref = None
        _servers[self.key] = self

    def matches(self, center, domega):
        """True when (center, domega) are the server's grid constants.  The
        same immutable objects (a tuple, a read-only array -- what
        energy._grid_constants hands out) are recognised by identity after
        the first byte-exact comparison."""
        if center is self._c_ref and domega is self._d_ref:
            return True
        d = self.W1.ndim
        cd = np.zeros(6)
        cd[:d], cd[3:3 + d] = center, domega
        if cd.tobytes() != self.cd_bytes:
            return False
        if _immutable(center) and _immutable(domega):
            self._c_ref, self._d_ref = center, domega
        return True

    def last_timing(self):
        """Timing of the last query in us (-1: not observed): host round trip,
        GPU detect -> result, post -> GPU detect, GPU result -> host receipt.
        A long round trip with a short GPU part locates the stall on the host
        or the PCIe path, not in the grid."""
        out = np.zeros(7)
        check(LIB.gf_server_last_timing(self.id, dptr(out)))
        return {"host_us": out[0], "gpu_us": out[1], "post_to_detect_us": out[2], "result_to_host_us": out[3],
                "post_us": out[4], "gpu_poll_gap_us": out[5], "gpu_clock_gap_us": out[6]}

    def retire(self):
        """The device side has exited (idle timeout): stop routing calls here."""
        if _servers.get(self.key) is self:
            del _servers[self.key]

    def stop(self):
        if self.id:
            if _servers.get(self.key) is self:
                del _servers[self.key]
            check(LIB.gf_server_stop(self.id))
            self.id = 0

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.stop()

    def __del__(self):
        try:
            self.stop()
        except Exception:
            pass


def pack_poses(R, t_eff):
    """(n, d, d) rotations + (n, d) effective translations -> (n, 12) float64."""
    R = np.asarray(R, dtype=np.float64)
    t = np.asarray(t_eff, dtype=np.float64)
    n, d = t.shape
    out = np.zeros((n, 12))
    if d == 3:
        out[:, :9] = R.reshape(n, 9)
        out[:, 9:] = t
    else:
        out[:, 0], out[:, 1], out[:, 3], out[:, 4] = R[:, 0, 0], R[:, 0, 1], R[:, 1, 0], R[:, 1, 1]
        out[:, 8] = 1.0
        out[:, 9:11] = t
    return out


def cascade_batch(C1, C2, wrap, domega, dcell, center, poses, out=None, precision=None, stream=None,
                  serial=False):
    """Batched cascade over poses (torch CUDA float64 tensor (n, 12), see
    pack_poses).  Returns a (n, 14) float64 CUDA tensor: interleaved complex
    [S, Tx, Ty, Tz, Gx, Gy, Gz] (2D: the rotational term is column pair 6).

    serial=True issues one single-query launch per pose (the haptic loop);
    otherwise one launch covers all poses (the pose sweep)."""
    import torch

    W1, W2 = as_device_window(C1), as_device_window(C2)
    if not (poses.is_cuda and poses.dtype == torch.float64 and poses.is_contiguous()):
        raise ValueError("poses must be a contiguous float64 CUDA tensor of shape (n, 12)")
    n = poses.shape[0]
    if out is None:
        out = torch.empty((n, 14), dtype=torch.float64, device=poses.device)
    d = W1.ndim
    dom = np.zeros(3)
    dom[:d] = domega
    cen = np.zeros(3)
    cen[:d] = center
    st = stream if stream is not None else torch.cuda.current_stream(poses.device).cuda_stream
    fn = LIB.gf_cascade_serial if serial else LIB.gf_cascade_batch
    check(fn(W1.handle, W2.handle, int(bool(wrap)), dptr(dom), float(dcell), dptr(cen),
                               _prec_bits(precision), int(n), ctypes.c_void_p(poses.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
    return out


# ---------------------------------------------------------------------------
# density operators (backend.py:71-150 of the reference)


def _elements(solid):
    return solid.element_arrays()


def distance_batch(solid, P, threads=None):
    """Min distance from each row of P to the solid's boundary elements
    (exact point-element distance, float64, bit-identical to the reference)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    _lib.ensure_device()
    elems, _, _ = _elements(solid)
    out = np.empty(len(P))
    if len(P):
        check(LIB.gf_distance_winding(solid.dimension, dptr(elems), len(elems), dptr(P), len(P), dptr(out), None))
    return out


def winding_batch(solid, P, threads=None):
    """Exact winding number (sum of per-element subtended angles)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    _lib.ensure_device()
    elems, _, _ = _elements(solid)
    out = np.empty(len(P))
    if len(P):
        check(LIB.gf_distance_winding(solid.dimension, dptr(elems), len(elems), dptr(P), len(P), None, dptr(out)))
    return out


def sweep_batch(solid, P, xi_eff, sigma, gconst, max_angle, max_depth, eta_min, threads=None):
    """Adaptive skeletal quadrature I+ per point; (values, residuals, clamp count)."""
    P = np.ascontiguousarray(P, dtype=np.float64)
    xi_eff = np.ascontiguousarray(xi_eff, dtype=np.float64)
    _lib.ensure_device()
    elems, normals, measures = _elements(solid)
    out = np.empty(len(P), dtype=np.complex128)
    resid = np.zeros(len(P))
    clamps = np.zeros(len(P), dtype=np.int64)
    if len(P):
        check(LIB.gf_sweep(solid.dimension, dptr(elems), dptr(np.ascontiguousarray(normals)), dptr(measures),
                           len(elems), dptr(P), dptr(xi_eff), len(P), float(sigma), float(gconst),
                           float(max_angle), int(max_depth), float(eta_min), dptr(out.view(np.float64)),
                           dptr(resid), clamps.ctypes.data_as(_lib.c_i64p)))
    return out, resid, int(clamps.sum())


def affinity_grid(solid, grid, family, sigma, gconst, lam_in, lam_out, max_angle, max_depth, eta_floor):
    """The whole affinity pipeline on the grid nodes, device resident.

    Returns (values: CUDA complex128 tensor of grid.node_count, flags: CUDA
    uint8 tensor (bit0 excluded, bit1 unresolved, bit2 inside), stats
    (total clamps, worst residual, distance+winding seconds, sweep seconds))."""
    import torch

    dev = _lib.ensure_device()
    elems, normals, measures = _elements(solid)
    m = grid.node_count
    values = torch.empty(m, dtype=torch.complex128, device=f"cuda:{dev}")
    flags = torch.empty(m, dtype=torch.uint8, device=f"cuda:{dev}")
    stats = np.zeros(4)
    dims = (ctypes.c_int32 * 3)(*(list(grid.dims) + [1] * (3 - len(grid.dims))))
    origin = np.zeros(3)
    origin[:grid.dimension] = grid.origin
    st = torch.cuda.current_stream(values.device).cuda_stream
    check(LIB.gf_affinity_grid(grid.dimension, dptr(elems), dptr(np.ascontiguousarray(normals)), dptr(measures),
                               len(elems), dims, dptr(origin), float(grid.spacing), int(family), float(sigma),
                               float(gconst), float(lam_in), float(lam_out), float(max_angle), int(max_depth),
                               float(eta_floor), ctypes.c_void_p(values.data_ptr()),
                               ctypes.c_void_p(flags.data_ptr()), dptr(stats), ctypes.c_void_p(st)))
    return values, flags, (int(stats[0]), float(stats[1]), float(stats[2]), float(stats[3]))


def affinity_planes(solid, grid, plane0, nplanes, halo_lo, halo_hi, family, sigma, gconst, lam_in, lam_out, max_angle,
                    max_depth, eta_floor):
    """`affinity_grid` restricted to axis-0 planes [plane0, plane0 + nplanes)
    of `grid` (halo planes computed for the neighbour fill, not returned);
    bit-identical to the same planes of the whole-grid result."""
    import torch

    dev = _lib.ensure_device()
    elems, normals, measures = _elements(solid)
    plane = int(np.prod(grid.dims[1:]))
    m = int(nplanes) * plane
    values = torch.empty(m, dtype=torch.complex128, device=f"cuda:{dev}")
    flags = torch.empty(m, dtype=torch.uint8, device=f"cuda:{dev}")
    stats = np.zeros(4)
    dims = (ctypes.c_int32 * 3)(*(list(grid.dims) + [1] * (3 - len(grid.dims))))
    origin = np.zeros(3)
    origin[:grid.dimension] = grid.origin
    st = torch.cuda.current_stream(values.device).cuda_stream
    check(LIB.gf_affinity_planes(grid.dimension, dptr(elems), dptr(np.ascontiguousarray(normals)), dptr(measures),
                                 len(elems), dims, dptr(origin), float(grid.spacing), int(plane0), int(nplanes),
                                 int(halo_lo), int(halo_hi), int(family), float(sigma), float(gconst), float(lam_in),
                                 float(lam_out), float(max_angle), int(max_depth), float(eta_floor),
                                 ctypes.c_void_p(values.data_ptr()), ctypes.c_void_p(flags.data_ptr()), dptr(stats),
                                 ctypes.c_void_p(st)))
    return values, flags, (int(stats[0]), float(stats[1]), float(stats[2]), float(stats[3]))


def winding_grid(solid, grid):
    """Winding numbers at every grid node as a CUDA float64 tensor (no host
    node-coordinate array; the kernel forms origin + h i itself)."""
    import torch

    dev = _lib.ensure_device()
    elems, _, _ = _elements(solid)
    out = torch.empty(grid.node_count, dtype=torch.float64, device=f"cuda:{dev}")
    dims = (ctypes.c_int32 * 3)(*(list(grid.dims) + [1] * (3 - len(grid.dims))))
    origin = np.zeros(3)
    origin[:grid.dimension] = grid.origin
    st = torch.cuda.current_stream(out.device).cuda_stream
    check(LIB.gf_winding_grid(grid.dimension, dptr(elems), len(elems), dims, dptr(origin), float(grid.spacing),
                              ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
    return out
