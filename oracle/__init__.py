"""CPU oracle for the geofield hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
``--impl reference`` arm) may import this package, and only as the checker.
The product package ``paper_1711_05017_b200`` never imports it.

Two layers:

* ``liboracle.so`` (oracle/geofield_oracle.c): a plain-C float64 restatement
  of the reference's compiled kernels (/root/reference/pkg/src/geofield/
  _core.pyx) -- cascade_2d/3d, distance, winding, sweep_2d/3d.
* numpy restatements of the reference's Python-level hot-path functions:
  the DFT convention and centred window (spectral.py:103-195), the
  multilinear window sampler (_fallback.py:312-351), the landscape
  (energy.py:309-344), the wrap mask (energy.py:278-306), the neighbour fill
  and the affinity combine (descriptor.py:283-357), the BVH builder
  (solids.py:297-343) and the bench pose generator (cli.py:51-70,336-346).

Parity of the oracle itself is pinned by tests/test_oracle_golden.py against
(a) ``oracle/_ref``: the reference's own Cython kernels compiled from the
sources under /root/reference by ``make -C oracle ref``, and (b) golden
fixtures in tests/golden/ produced by tests/golden/make_golden.py, which
imports the unmodified reference package.
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import itertools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


def lib():
    """Load oracle/liboracle.so (built by ``make -C oracle``)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing; run `make -C oracle`")
        L = ctypes.CDLL(path)
        L.orc_cascade_3d.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                     _dp, _dp, _dp, _dp]
        L.orc_cascade_2d.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp, _dp, _dp, _dp]
        L.orc_distance_brute.argtypes = [ctypes.c_int, _dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp]
        L.orc_distance.argtypes = [ctypes.c_int, _dp, _dp, _ip, _ip, _ip, _ip, _ip, _dp, _dp,
                                   ctypes.c_int64, _dp]
        L.orc_winding.argtypes = [ctypes.c_int, _dp, ctypes.c_int64, _dp, ctypes.c_int64, _dp]
        sweep_args = [_dp, _dp, _dp, ctypes.c_int64, _dp, _dp, ctypes.c_int64, ctypes.c_double,
                      ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double, _dp, _dp, _ip]
        L.orc_sweep_3d.argtypes = sweep_args
        L.orc_sweep_2d.argtypes = sweep_args
        _LIB = L
    return _LIB


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


# ---------------------------------------------------------------------------
# compiled kernels (C restatement of _core.pyx)


def cascade(C1, C2, wrap, domega, dcell, R, t_eff, center):
    """backend.cascade contract (backend.py:153-164) on the C restatement."""
    C1, C2 = _c128(C1), _c128(C2)
    R, t_eff, center = _f64(R), _f64(t_eff), _f64(center)
    if C1.ndim == 3:
        out = np.empty(7, dtype=np.complex128)
        lib().orc_cascade_3d(_d(C1.view(np.float64)), _d(C2.view(np.float64)), *C1.shape, int(bool(wrap)),
                             float(domega[0]), float(domega[1]), float(domega[2]), float(dcell),
                             _d(R), _d(t_eff), _d(center), _d(out.view(np.float64)))
    else:
        out = np.empty(4, dtype=np.complex128)
        lib().orc_cascade_2d(_d(C1.view(np.float64)), _d(C2.view(np.float64)), *C1.shape, int(bool(wrap)),
                             float(domega[0]), float(domega[1]), float(dcell),
                             _d(R), _d(t_eff), _d(center), _d(out.view(np.float64)))
    return out


def _elements(elems):
    """Triangles ((n, 3, 3) or flat (n, 9)) -> d = 3; segments ((n, 2, 2) or (n, 4)) -> d = 2."""
    e = _f64(elems)
    e = e.reshape(len(e), -1)
    if e.shape[1] == 9:
        return e, 3
    if e.shape[1] == 4:
        return e, 2
    raise ValueError("elements must be triangles (n, 9) or segments (n, 4)")


def _rows(m, fn, min_rows=256):
    """Run fn(i0, i1) over [0, m) in row blocks on every host core (the C
    kernels release nothing shared; ctypes drops the GIL).  Per-point
    results do not depend on the split."""
    from concurrent.futures import ThreadPoolExecutor

    nt = max(1, min(os.cpu_count() or 1, m // min_rows))
    if nt == 1:
        fn(0, m)
        return
    bounds = np.linspace(0, m, 4 * nt + 1).astype(np.int64)
    with ThreadPoolExecutor(max_workers=nt) as pool:
        list(pool.map(lambda k: fn(int(bounds[k]), int(bounds[k + 1])), range(len(bounds) - 1)))


def _at(a, i0):
    """ctypes pointer to row i0 of a C-contiguous float64 / int64 array."""
    return ctypes.cast(a.ctypes.data + i0 * a.strides[0], _ip if a.dtype == np.int64 else _dp)


def distance(elems, P):
    """Exact min point-element distance (triangles (n,3,3) or segments (n,2,2))."""
    e, d = _elements(elems)
    P = _f64(P)
    out = np.empty(len(P))
    _rows(len(P), lambda i0, i1: lib().orc_distance_brute(d, _d(e), len(e), _at(P, i0), i1 - i0, _at(out, i0)))
    return out


def distance_bvh(bvh, elems, P):
    """Same, by the reference's BVH stack traversal (_core.pyx:189-230)."""
    e, d = _elements(elems)
    P = _f64(P)
    bmin, bmax, left, right, start, count, perm = bvh
    ints = [np.ascontiguousarray(x, dtype=np.int64) for x in (left, right, start, count, perm)]
    out = np.empty(len(P))
    lib().orc_distance(d, _d(_f64(bmin)), _d(_f64(bmax)), *[_i(x) for x in ints], _d(e), _d(P), len(P),
                       _d(out))
    return out


def winding(elems, P):
    e, d = _elements(elems)
    P = _f64(P)
    out = np.empty(len(P))
    _rows(len(P), lambda i0, i1: lib().orc_winding(d, _d(e), len(e), _at(P, i0), i1 - i0, _at(out, i0)))
    return out


def sweep(elems, normals, measures, P, xi_eff, sigma, gconst, max_angle, max_depth, eta_min):
    """Adaptive skeletal sweep; returns (I+ complex128, resid, clamps int)."""
    e, d = _elements(elems)
    P, xi_eff = _f64(P), _f64(xi_eff)
    normals, measures = _f64(normals), _f64(measures)
    out = np.empty(len(P), dtype=np.complex128)
    resid = np.zeros(len(P))
    clamps = np.zeros(len(P), dtype=np.int64)
    fn = lib().orc_sweep_3d if d == 3 else lib().orc_sweep_2d
    o64 = out.view(np.float64).reshape(len(P), 2)
    _rows(len(P), lambda i0, i1: fn(_d(e), _d(normals), _d(measures), len(e), _at(P, i0), _at(xi_eff, i0), i1 - i0,
                                    float(sigma), float(gconst), float(max_angle), int(max_depth), float(eta_min),
                                    _at(o64, i0), _at(resid, i0), _at(clamps, i0)))
    return out, resid, int(clamps.sum())


# ---------------------------------------------------------------------------
# the reference's own compiled kernels (oracle/_ref, built from /root/reference)


def ref_core():
    """Import oracle/_ref/_core*.so, or return None if it was not built."""
    hits = glob.glob(os.path.join(_HERE, "_ref", "_core*.so"))
    if not hits:
        return None
    spec = importlib.util.spec_from_file_location("_core", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


# ---------------------------------------------------------------------------
# grid helpers (descriptor.py:111-173)


def grid_points(dims, origin, spacing):
    axes = [origin[a] + spacing * np.arange(dims[a]) for a in range(len(dims))]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([g.ravel() for g in mesh], axis=1)


def grid_center(dims, origin, spacing):
    return np.asarray([origin[a] + spacing * (dims[a] // 2) for a in range(len(dims))])


def window_freqs(window, domega):
    """spectral.py:176-181"""
    axes = [(np.arange(w) - w // 2) * dw for w, dw in zip(window, domega)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([g.ravel() for g in mesh], axis=1)


# ---------------------------------------------------------------------------
# spectral restatement (spectral.py:103-195)


def forward_dft(values, dims, origin, spacing):
    """A(w) = dV fftshift(fftn(f)) prod_a exp(-2 pi i w_a o_a), DC-centred."""
    d = len(dims)
    F = np.fft.fftshift(np.fft.fftn(np.asarray(values).reshape(dims))) * spacing ** d
    for a in range(d):
        freqs = np.fft.fftshift(np.fft.fftfreq(dims[a], d=spacing))
        shape = [1] * d
        shape[a] = dims[a]
        F = F * np.exp(-2j * np.pi * freqs * origin[a]).reshape(shape)
    return F


def center_window(A, dims, origin, spacing, w=None):
    """Centred slice of side w (None = full) times exp(+2 pi i w.c)."""
    d = len(dims)
    if w is None or w == dims[0]:
        win = tuple(dims)
        amps = A
    else:
        win = (w,) * d
        amps = A[tuple(slice(n // 2 - w // 2, n // 2 + w // 2) for n in dims)]
    dom = [1.0 / (n * spacing) for n in dims]
    W = window_freqs(win, dom)
    phase = np.exp(2j * np.pi * (W @ grid_center(dims, origin, spacing))).reshape(win)
    return amps * phase


def interp_window(C, u, wrap):
    """Multilinear sample + index gradient, zero outside unless wrap (_fallback.py:312-351)."""
    d = C.ndim
    dims = C.shape
    flat = C.ravel()
    i0 = np.floor(u).astype(np.int64)
    f = u - i0
    M = len(u)
    V = np.zeros(M, dtype=np.complex128)
    dV = np.zeros((M, d), dtype=np.complex128)
    for corner in itertools.product((0, 1), repeat=d):
        idx = i0 + np.asarray(corner, dtype=np.int64)
        lin = np.zeros(M, dtype=np.int64)
        if wrap:
            for a in range(d):
                lin = lin * dims[a] + idx[:, a] % dims[a]
            cv = flat[lin]
        else:
            ok = np.ones(M, dtype=bool)
            for a in range(d):
                ok &= (idx[:, a] >= 0) & (idx[:, a] < dims[a])
                lin = lin * dims[a] + np.clip(idx[:, a], 0, dims[a] - 1)
            cv = np.where(ok, flat[lin], 0.0)
        wgt = np.ones(M)
        for a in range(d):
            wgt = wgt * (f[:, a] if corner[a] else 1.0 - f[:, a])
        V += wgt * cv
        for a in range(d):
            dw = np.ones(M)
            for b in range(d):
                if b != a:
                    dw = dw * (f[:, b] if corner[b] else 1.0 - f[:, b])
            dV[:, a] += (dw if corner[a] else -dw) * cv
    return V, dV


def score_field(C1, C2, wrap, dims, origin, spacing, R):
    """Landscape over node translations (energy.py:309-344), values only."""
    d = len(dims)
    window = C1.shape
    dom = np.asarray([1.0 / (n * spacing) for n in dims])
    W = window_freqs(window, dom)
    u = -(W @ R) / dom + np.asarray([w // 2 for w in window])
    V, _ = interp_window(C2, u, wrap)
    c = grid_center(dims, origin, spacing)
    Q = (C1.ravel() * V * np.exp(2j * np.pi * (W @ (R @ c - c)))).reshape(window)
    full = np.zeros(dims, dtype=np.complex128)
    full[tuple(slice(n // 2 - w // 2, n // 2 + w // 2) for n, w in zip(dims, window))] = Q
    for a in range(d):
        freqs = np.fft.fftshift(np.fft.fftfreq(dims[a], d=spacing))
        shape = [1] * d
        shape[a] = dims[a]
        full = full * np.exp(2j * np.pi * freqs * origin[a]).reshape(shape)
    return np.fft.ifftn(np.fft.ifftshift(full)) / spacing ** d


def rotated_box(lo, hi, R):
    """energy.py:278-283"""
    d = len(lo)
    corners = np.stack(np.meshgrid(*[(lo[a], hi[a]) for a in range(d)], indexing="ij"), axis=-1)
    corners = corners.reshape(-1, d) @ R.T
    return corners.min(axis=0), corners.max(axis=0)


def wrap_mask(dims, origin, spacing, box1, box2, R):
    """energy.py:286-306 (box1/box2 = (lo, hi) solid boxes, or None)."""
    d = len(dims)
    if box1 is None or box2 is None:
        return np.zeros(dims, dtype=bool)
    glo = np.asarray(origin) - 0.5 * spacing
    ghi = glo + spacing * np.asarray(dims)
    rlo, rhi = rotated_box(np.asarray(box2[0], float), np.asarray(box2[1], float), R)
    r1 = 0.5 * float(np.linalg.norm(np.asarray(box1[1], float) - np.asarray(box1[0], float)))
    lo_ok = glo + r1 - rlo
    hi_ok = ghi - r1 - rhi
    mask = np.zeros(dims, dtype=bool)
    for a in range(d):
        ax = origin[a] + spacing * np.arange(dims[a])
        shape = [1] * d
        shape[a] = dims[a]
        mask |= ((ax < lo_ok[a]) | (ax > hi_ok[a])).reshape(shape)
    return mask


# ---------------------------------------------------------------------------
# density restatement (descriptor.py:283-357)


def neighbor_average(values, excluded, dims):
    """Excluded nodes take the mean of their non-excluded face neighbours."""
    vals = values.reshape(dims)
    ex = excluded.reshape(dims)
    acc = np.zeros(dims, dtype=np.complex128)
    cnt = np.zeros(dims, dtype=np.int64)
    d = len(dims)
    for a in range(d):
        for off in (-1, 1):
            src = [slice(None)] * d
            dst = [slice(None)] * d
            src[a], dst[a] = (slice(1, None), slice(0, -1)) if off == 1 else (slice(0, -1), slice(1, None))
            good = ~ex[tuple(src)]
            acc[tuple(dst)] += np.where(good, vals[tuple(src)], 0)
            cnt[tuple(dst)] += good
    with np.errstate(invalid="ignore"):
        avg = np.where(cnt > 0, acc / np.maximum(cnt, 1), 0)
    return np.where(ex, avg, vals).ravel()


def affinity_values(elems, normals, measures, dims, origin, spacing, sigma=0.5, lambda_in=1.0,
                    lambda_out=3.0, max_angle=0.02, max_depth=16, eta_floor=0.25, family="SkeletalDensity"):
    """The whole affinity_field pipeline on the C restatement.

    Returns (values complex128, flags list, stats dict, xi, wind)."""
    d = len(dims)
    eta_min = eta_floor * spacing
    P = grid_points(dims, origin, spacing)
    xi = distance(elems, P)
    wind = winding(elems, P)
    inside = wind >= 0.5
    excluded = xi < eta_min
    if family == "InverseSquare":
        values = wind.astype(np.complex128)
        resid = np.zeros(len(P))
        nclamp = 0
    else:
        gconst = 1.0 / (4.0 * np.pi) if d == 3 else 1.0 / (2.0 * np.pi)
        iplus, resid, nclamp = sweep(elems, normals, measures, P, np.maximum(xi, eta_min), sigma, gconst,
                                     max_angle, max_depth, eta_min)
        values = np.where(inside, lambda_in * np.conj(iplus), -lambda_out * iplus)
    values = neighbor_average(values, excluded, dims)
    unresolved = np.nonzero(resid > max_angle)[0]
    stats = dict(excluded=int(excluded.sum()), eta_clamped=int(nclamp),
                 worst_residual=float(resid.max()) if len(resid) else 0.0,
                 unresolved_nodes=len(unresolved), inside_nodes=int(inside.sum()))
    flags = sorted(set(np.nonzero(excluded)[0].tolist()) | set(unresolved.tolist()))
    return values, flags, stats, xi, wind


# ---------------------------------------------------------------------------
# bench pose generator (cli.py:51-70, 336-346), bit-identical draw order


def quat_rotation(q):
    w, x, y, z = [float(v) for v in q]
    n = np.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def bench_poses(n, span, seed=0):
    rng = np.random.default_rng(seed)
    Rs, ts = [], []
    for _ in range(n):
        q = rng.normal(size=4)
        Rs.append(quat_rotation([float(str(v)) for v in q]))
        ts.append(rng.uniform(-span, span, 3))
    return np.asarray(Rs), np.asarray(ts)


def cascade_term_scales(C1, C2, wrap, domega, dcell, R, t_eff, center):
    """Per-output L1 scale dcell * sum |summand| of the cascade (the
    denominator floor of the parity tolerance);
    numpy restatement of _fallback.cascade_eval (_fallback.py:364-391)."""
    C1, C2 = np.asarray(C1), np.asarray(C2)
    d = C1.ndim
    win = C1.shape
    W = window_freqs(win, domega)
    u = -(W @ R) / np.asarray(domega) + np.asarray([w // 2 for w in win])
    V, dV = interp_window(C2, u, wrap)
    base = C1.ravel() * np.exp(2j * np.pi * (W @ t_eff))
    out = [np.sum(np.abs(base * V))]
    for a in range(d):
        out.append(np.sum(np.abs(base * V * 2 * np.pi * W[:, a])))
    gens = [np.array([[0.0, -1.0], [1.0, 0.0]])] if d == 2 else [
        np.array([[0.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]]),
        np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 0.0], [-1.0, 0.0, 0.0]]),
        np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])]
    dVn = dV / np.asarray(domega)
    for G in gens:
        dnu = -(W @ (G @ R))
        t1 = np.einsum("ij,ij->i", dVn, dnu)
        t2 = 2j * np.pi * (W @ (G @ (R @ center))) * V
        out.append(np.sum(np.abs(base * t1)) + np.sum(np.abs(base * t2)))
    return dcell * np.asarray(out)


# ---------------------------------------------------------------------------
# Independent real-space / direct-sum references for the query and landscape
# (restating the reference's slow paths, /root/reference/pkg/src/geofield/
# oracle.py:30-136 and :224-275, in this package's own terms).


def node_interp(values, dims, origin, spacing, Q, wrap):
    """Multilinear interpolation of node values at physical points Q (m, d):
    zero outside the node box, or periodic when wrap (oracle.py:30-57)."""
    dims = tuple(dims)
    d = len(dims)
    vals = np.asarray(values).reshape(dims)
    u = (np.asarray(Q, dtype=np.float64) - np.asarray(origin, dtype=np.float64)) / spacing
    i0 = np.floor(u).astype(np.int64)
    fr = u - i0
    acc = np.zeros(len(u), dtype=np.complex128)
    for corner in np.ndindex(*(2,) * d):
        idx = i0 + np.asarray(corner)
        wgt = np.prod(np.where(np.asarray(corner) == 1, fr, 1.0 - fr), axis=1)
        if wrap:
            acc += wgt * vals[tuple((idx % np.asarray(dims)).T)]
        else:
            inside = np.all((idx >= 0) & (idx < np.asarray(dims)), axis=1)
            safe = np.where(inside[:, None], idx, 0)
            acc += np.where(inside, wgt * vals[tuple(safe.T)], 0.0)
    return acc


def brute_score(v1, v2, dims, origin, spacing, R, t, wrap=False):
    """sum_j rho1(p_j) rho2(R^T (p_j - t)) dV over the grid nodes
    (oracle.py:60-74)."""
    P = grid_points(dims, origin, spacing)
    Q = (P - np.asarray(t, dtype=np.float64)) @ np.asarray(R, dtype=np.float64)
    s = node_interp(v2, dims, origin, spacing, Q, wrap)
    return complex(np.sum(np.asarray(v1).ravel() * s) * spacing ** len(dims))


def direct_amplitudes(values, dims, origin, spacing, W):
    """A(w) = sum_i f_i exp(-2 pi i w.p_i) dV at arbitrary frequencies W (k, d)
    by explicit summation (oracle.py:85-93)."""
    P = grid_points(dims, origin, spacing)
    f = np.asarray(values).ravel()
    dV = spacing ** len(dims)
    return np.array([np.sum(f * np.exp(-2j * np.pi * (P @ w))) * dV for w in np.asarray(W)])


def cascade_direct(v1, v2, dims, origin, spacing, R, t, side=None):
    """Mode sum with exactly rotated amplitudes (no interpolation): the
    band-limited score over the centred window of `side` modes per axis
    (oracle.py:105-136)."""
    dims = tuple(dims)
    d = len(dims)
    dom = np.array([1.0 / (n * spacing) for n in dims])
    sides = dims if side is None else (side,) * d
    W = window_freqs(sides, dom)
    A1 = direct_amplitudes(v1, dims, origin, spacing, W)
    A2 = direct_amplitudes(v2, dims, origin, spacing, -(W @ np.asarray(R, dtype=np.float64)))
    dcell = 1.0 / (np.prod(dims) * spacing ** d)
    return complex(np.sum(A1 * A2 * np.exp(2j * np.pi * (W @ np.asarray(t, dtype=np.float64)))) * dcell)


def axis_rotation(d, axis, angle):
    if d == 2:
        c, s = np.cos(angle), np.sin(angle)
        return np.array([[c, -s], [s, c]])
    k = np.zeros(3)
    k[axis] = 1.0
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * (K @ K)


def fd_gradient(scorer, R, t, dt=1e-6, dr=1e-6):
    """Central differences of scorer(R, t): translation components, then the
    left-multiplied rotation generators, with the rotation step refined until
    two estimates agree (oracle.py:234-275)."""
    R = np.asarray(R, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    d = len(t)
    tg = np.empty(d, dtype=np.complex128)
    for a in range(d):
        e = np.zeros(d)
        e[a] = dt
        tg[a] = (scorer(R, t + e) - scorer(R, t - e)) / (2 * dt)
    n_rot = 1 if d == 2 else 3
    rg = np.empty(n_rot, dtype=np.complex128)
    for g in range(n_rot):
        step = dr
        est = (scorer(axis_rotation(d, g, step) @ R, t) - scorer(axis_rotation(d, g, -step) @ R, t)) / (2 * step)
        for _ in range(3):
            step /= 10.0
            finer = (scorer(axis_rotation(d, g, step) @ R, t) - scorer(axis_rotation(d, g, -step) @ R, t)) / (2 * step)
            done = abs(finer - est) <= 1e-4 * max(abs(finer), 1e-12)
            est = finer
            if done:
                break
        rg[g] = est
    return tg, rg


def disk_density(sigma, lam_in, lam_out, a, radii, n_theta=2048):
    """Skeletal density of a disk of radius a at distance r from its centre by
    Gauss-Legendre quadrature of the one angular boundary integral -- an
    independent route to the swept density (oracle.py:278-318): interior
    points take lam_in * conj(I), exterior -lam_out * I."""
    x, wts = np.polynomial.legendre.leggauss(n_theta)
    th = np.pi * (x + 1.0)
    wq = np.pi * wts
    qx, qy = a * np.cos(th), a * np.sin(th)
    out = []
    for r in np.atleast_1d(radii):
        xi = abs(r - a)
        rx, ry = qx - r, qy
        eta = np.hypot(rx, ry)
        proj = (qx * rx + qy * ry) / (a * eta)
        g = np.exp(-0.5 * ((eta / xi - 1.0) / sigma) ** 2) / (np.sqrt(2.0 * np.pi) * sigma)
        z = xi + 1j * eta
        I = np.sum(wq * g * proj / (z * z)) * a / (2.0 * np.pi)
        out.append(lam_in * np.conj(I) if r < a else -lam_out * I)
    return np.asarray(out)


def raycast_inside(triangles, P, seed=0):
    """Point-in-mesh by ray-crossing parity (an independent test of the
    winding classification; reference oracle.py:161-221): one random
    direction per batch, Moller-Trumbore hits, and points whose ray grazes an
    edge or vertex (barycentric within 1e-9 of the boundary) are re-cast with
    a fresh direction."""
    tri = np.asarray(triangles, dtype=np.float64).reshape(-1, 3, 3)
    P = np.asarray(P, dtype=np.float64)
    rng = np.random.default_rng(seed)
    out = np.zeros(len(P), dtype=bool)
    todo = np.arange(len(P))
    a, e1, e2 = tri[:, 0], tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]
    while len(todo):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        pv = np.cross(d, e2)                      # (n, 3)
        det = np.einsum("ij,ij->i", e1, pv)
        ok_det = np.abs(det) > 1e-14
        inv = np.where(ok_det, 1.0 / np.where(ok_det, det, 1.0), 0.0)
        graze = np.zeros(len(todo), dtype=bool)
        count = np.zeros(len(todo), dtype=np.int64)
        for c0 in range(0, len(todo), 512):
            idx = todo[c0:c0 + 512]
            s = P[idx][:, None, :] - a[None, :, :]   # (m, n, 3)
            u = np.einsum("mnk,nk->mn", s, pv) * inv
            q = np.cross(s, e1[None, :, :])
            v = np.einsum("k,mnk->mn", d, q) * inv
            t = np.einsum("nk,mnk->mn", e2, q) * inv
            hit = ok_det & (u >= 0) & (v >= 0) & (u + v <= 1) & (t > 0)
            near = ok_det & (t > 0) & ((np.abs(u) < 1e-9) | (np.abs(v) < 1e-9) | (np.abs(u + v - 1) < 1e-9)) & \
                (u > -1e-9) & (v > -1e-9) & (u + v < 1 + 1e-9)
            count[c0:c0 + 512] = hit.sum(axis=1)
            graze[c0:c0 + 512] = near.any(axis=1)
        done = ~graze
        out[todo[done]] = (count[done] % 2) == 1
        todo = todo[graze]
    return out


def _interp_values(C, u, wrap):
    """V only of interp_window (no index gradient): the multilinear sample."""
    d = C.ndim
    dims = C.shape
    flat = C.ravel()
    i0 = np.floor(u).astype(np.int64)
    f = u - i0
    V = np.zeros(len(u), dtype=np.complex128)
    for corner in itertools.product((0, 1), repeat=d):
        lin = np.zeros(len(u), dtype=np.int64)
        ok = np.ones(len(u), dtype=bool)
        wgt = np.ones(len(u))
        for a in range(d):
            ia = i0[:, a] + corner[a]
            if wrap:
                ia = ia % dims[a]
            else:
                ok &= (ia >= 0) & (ia < dims[a])
                ia = np.clip(ia, 0, dims[a] - 1)
            lin = lin * dims[a] + ia
            wgt = wgt * (f[:, a] if corner[a] else 1.0 - f[:, a])
        V += np.where(ok, wgt * flat[lin], 0.0)
    return V


def score_field_scale(C1, C2, wrap, dims, spacing, R, stride=1, chunk=1 << 22):
    """dcell * sum_w |C1(w) V(w)|: the L1 floor of the landscape parity
    tolerance (the translation phase has unit modulus, so it is the same at
    every voxel; energy.py:309-344).  Modes are taken in x-plane chunks so a
    512^3 window stays within a few GB; stride > 1 estimates the sum from
    every stride-th mode per axis (times stride^d)."""
    C1 = np.asarray(C1)
    window = C1.shape
    d = len(window)
    dom = np.asarray([1.0 / (n * spacing) for n in dims])
    half = np.asarray([w // 2 for w in window])
    ks = [np.arange(0, w, stride) for w in window]
    total = 0.0
    per = max(1, chunk // int(np.prod([len(k) for k in ks[1:]])))
    for x0 in range(0, len(ks[0]), per):
        kk = [ks[0][x0:x0 + per]] + ks[1:]
        mesh = np.meshgrid(*kk, indexing="ij")
        K = np.stack([m.ravel() for m in mesh], axis=1)
        W = (K - half) * dom
        V = _interp_values(C2, -(W @ R) / dom + half, wrap)
        total += float(np.sum(np.abs(C1[tuple(mesh)].ravel() * V)))
    dcell = 1.0 / (float(np.prod(dims)) * spacing ** d)
    return dcell * total * stride ** d


def rotational_gradient_vector(C1, C2, moments, wrap, domega, dcell, R, t, center):
    """Moment-spectrum rotational gradient: numpy restatement of
    energy._rotational_gradient_vector (energy.py:210-251), the reference's
    cross-check of the torque; `moments` are the centre-referenced windows
    of rho p_a, `t` the configuration translation."""
    C1 = np.asarray(C1)
    d = C1.ndim
    window = C1.shape
    dom = np.asarray(domega, dtype=np.float64)
    W = window_freqs(window, dom)
    u = -(W @ R) / dom + np.asarray([w // 2 for w in window])
    V, _ = interp_window(np.asarray(C2), u, wrap)
    c = np.asarray(center, dtype=np.float64)
    M = [-(interp_window(np.asarray(mw), u, wrap)[0]) + c[a] * V for a, mw in enumerate(moments)]
    t_eff = np.asarray(t, dtype=np.float64) - c + R @ c
    base = C1.ravel() * np.exp(2j * np.pi * (W @ t_eff))
    gens = [np.array([[0.0, -1.0], [1.0, 0.0]])] if d == 2 else [
        np.array([[0.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]]),
        np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 0.0], [-1.0, 0.0, 0.0]]),
        np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])]
    out = []
    for G in gens:
        dirs = W @ (R.T @ G).T
        samp = sum(dirs[:, a] * M[a] for a in range(d))
        out.append(dcell * (2j * np.pi * np.sum(base * samp) + 2j * np.pi * np.sum(base * (W @ (G @ (R @ c))) * V)))
    return np.asarray(out)
