"""Multi-GPU paths: one process per GPU.

* Pose sweep (Q3): poses are independent units -> contiguous pose ranges per
  rank, no collective in the loop; results are optionally all-gathered once.
  The reference has no sweep (it loops evaluate() serially, cli.py:349-356).
* Landscape (F1) at large N: slab decomposition with one exchange step.
  Rank r owns window x-planes [a_r, b_r): it forms its Q planes (product
  kernel restricted to those planes) and runs the two inner inverse passes
  (z then y: w -> N), giving (b_r - a_r, N1, N2).  An all-to-all re-slices
  the data by output y-slabs (each rank gets every x-plane of its y-range),
  and the last pass inverts along x (w0 -> N0).  Rank r ends with the
  landscape rows y in [c_r, d_r): an (N0, d_r - c_r, N2) slab.
* Forward window (W1) of a node-sharded field: the z pass runs on each
  rank's x-planes, the y pass (pruned N -> w) stores straight into the
  window y-slabs of the destination ranks (NCCL: symmetric memory; gloo: an
  all-to-all after the pass), and the x pass (N0 -> w) finishes; only the
  (2K)^3 window ever crosses the fabric.
* Density (D1/D2): node slabs along axis 0, one per rank, triangles
  replicated; each rank also computes one halo plane per interior side so
  the excluded-node neighbour fill is exact across slab boundaries (the
  halo is computed, not exchanged: no collective on the data path).  Counts
  and flags are reduced once at the end.
* The single haptic query does not shard: replicas only.

The decomposition logic (ranges, split sizes, re-assembly) is host code that
runs the same with NCCL on GPUs and gloo on CPUs; `tests/test_parallel.py`
drives it with gloo at world size 2.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, backend


def shard_range(n, rank, world):
    """Contiguous [lo, hi) share of n units for `rank` (balanced to +-1)."""
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist

    return dist


def _world(group):
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


# ---------------------------------------------------------------------------
# pose sweep


def gather_rows(local, n_total, group=None):
    """All-gather per-rank row blocks (contiguous shard_range layout) into
    the full (n_total, ...) array on every rank; works for NCCL and gloo."""
    import torch

    rank, world = _world(group)
    if world == 1:
        return local
    dist = _dist()
    rows = [shard_range(n_total, r, world) for r in range(world)]
    width = max(hi - lo for lo, hi in rows)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: hi - lo] for b, (lo, hi) in zip(bufs, rows)], dim=0)


def pose_sweep(asset1, asset2, rotations, translations, m_prime=None, precision=None, group=None, gather=True,
               compute=None):
    """Evaluate many poses, sharded by pose across the ranks of `group`.

    rotations (n, d, d), translations (n, d) (host arrays, the same on every
    rank).  Returns a (n, 7) complex128 host array [S, T..., G...] (2D: 4
    columns) when gather, else this rank's (hi - lo, 7) shard and its range.
    `compute(asset1, asset2, R_shard, t_shard)` may replace the GPU kernel
    (tests run the decomposition on CPU with the oracle)."""
    import torch

    rank, world = _world(group)
    R = np.asarray(rotations, dtype=np.float64)
    t = np.asarray(translations, dtype=np.float64)
    n = len(t)
    lo, hi = shard_range(n, rank, world)
    if compute is None:
        local = _sweep_gpu(asset1, asset2, R[lo:hi], t[lo:hi], m_prime, precision)
    else:
        local = torch.as_tensor(compute(asset1, asset2, R[lo:hi], t[lo:hi]))
    if not gather:
        return local.cpu().numpy(), (lo, hi)
    full = gather_rows(torch.view_as_real(local.contiguous()) if local.is_complex() else local, n, group)
    if not full.is_complex():
        full = torch.view_as_complex(full.contiguous())
    return full.cpu().numpy()


def _sweep_gpu(asset1, asset2, R, t, m_prime, precision):
    """Local shard through the batched cascade kernel; (k, 7) complex128 CUDA tensor."""
    import torch

    g = asset1.grid
    c = g.center()
    C1, wrap1 = asset1.window(m_prime)
    C2, wrap2 = asset2.window(m_prime)
    t_eff = t - c + np.einsum("nij,j->ni", R, c) if len(t) else t
    poses = torch.from_numpy(backend.pack_poses(R, t_eff)).to(f"cuda:{_lib.ensure_device()}")
    dcell = 1.0 / (g.node_count * g.cell_volume)
    out = backend.cascade_batch(C1, C2, wrap1 and wrap2, g.delta_omega(), dcell, c, poses, precision=precision)
    res = torch.view_as_complex(out.reshape(-1, 7, 2))
    if g.dimension == 2:
        res = res[:, [0, 1, 2, 6]]
    return res


# ---------------------------------------------------------------------------
# slab-decomposed landscape


def slab_plan(window, dims, world):
    """Per-rank window x-plane ranges and output y-slab ranges."""
    kx = [shard_range(window[0], r, world) for r in range(world)]
    ys = [shard_range(dims[1], r, world) for r in range(world)]
    return kx, ys


def exchange_planes_to_slabs(local, kx_ranges, y_ranges, rank, group=None):
    """All-to-all: local (nk_r, N1, N2) x-planes -> (w0, ny_r, N2) y-slab.

    Works on real tensors (complex data travels as view_as_real)."""
    import torch

    dist = _dist()
    world = len(kx_ranges)
    nk = local.shape[0]
    tail = tuple(local.shape[2:])
    send = torch.cat([local[:, lo:hi].reshape(-1) for lo, hi in y_ranges])
    in_splits = [nk * (hi - lo) * int(np.prod(tail)) for lo, hi in y_ranges]
    ny = y_ranges[rank][1] - y_ranges[rank][0]
    out_splits = [(khi - klo) * ny * int(np.prod(tail)) for klo, khi in kx_ranges]
    recv = torch.empty(sum(out_splits), dtype=local.dtype, device=local.device)
    if world == 1:
        recv.copy_(send)
    else:
        dist.all_to_all_single(recv, send, out_splits, in_splits, group=group)
    parts = torch.split(recv, out_splits)
    blocks = [p.reshape((khi - klo, ny) + tail) for p, (klo, khi) in zip(parts, kx_ranges)]
    return torch.cat(blocks, dim=0)


_SYMM = {}


def _symm_slab(shape, dtype, group):
    """Symmetric-memory slab buffer (same size on every rank) and its
    handle; cached per (shape, dtype, group)."""
    import torch
    import torch.distributed._symmetric_memory as symm_mem

    dist = _dist()
    g = group or dist.group.WORLD
    key = (tuple(shape), dtype, id(g))
    if key not in _SYMM:
        real = torch.float64 if dtype == torch.complex128 else torch.float32
        buf = symm_mem.empty(*shape, 2, dtype=real, device=f"cuda:{_lib.ensure_device()}")
        _SYMM[key] = (buf, symm_mem.rendezvous(buf, g))
    return _SYMM[key]


def scatter_y_pass(a, n1, bounds, dst_ptrs, x_off, precision, forward=False):
    """An axis-1 pass of this rank's planes `a` (nk, L1, N2) stored straight
    into the destination ranks' y-slabs (gf_fft_pass_scatter).  Inverse
    (landscape): centred window in, n1 node rows out.  forward=True (window):
    node rows in, the centred window of bounds[-1] rows out with the (-1)^m
    centre phase, as spectral.forward_window."""
    import torch

    si = (ctypes.c_int32 * 3)(*a.shape)
    yb = (ctypes.c_int32 * len(bounds))(*bounds)
    dp = (ctypes.c_uint64 * len(dst_ptrs))(*dst_ptrs)
    st = torch.cuda.current_stream(a.device).cuda_stream
    if forward:
        args = (0, int(bounds[-1]), 1, -1, 0.0, 0.5)
    else:
        args = (1, int(n1), 0, 1, 0.0, 0.0)
    _lib.check(_lib.LIB.gf_fft_pass_scatter(precision, ctypes.c_void_p(a.data_ptr()), si, int(n1), *args, 1.0,
                                            len(dst_ptrs), yb, dp, int(x_off), ctypes.c_void_p(st)))


def score_field_slab(asset1, asset2, R, m_prime=None, precision=64, group=None, exchange="auto"):
    """This rank's y-slab (N0, ny, N2) of the landscape (energy.score_field),
    as a CUDA complex tensor.  Gather the slabs along axis 1 for the full
    N^3 field.  The exchange between the inner passes and the x pass is
    either fused into the y pass (exchange="fused", the default on NCCL: the
    pass stores each line straight into its destination rank's symmetric-
    memory slab over NVLink, then one device-side barrier) or an
    all-to-all ("alltoall", the gloo path)."""
    import torch

    from .energy import _check_pair
    from .spectral import check_rotation

    _check_pair(asset1, asset2)
    g = asset1.grid
    if g.dimension != 3:
        raise ValueError("slab decomposition is for 3D landscapes")
    R = check_rotation(R, 3)
    rank, world = _world(group)
    C1, wrap1 = asset1.window(m_prime)
    C2, wrap2 = asset2.window(m_prime)
    wrap = wrap1 and wrap2
    w = list(C1.shape)
    N = list(g.dims)
    kx_r, y_r = slab_plan(w, N, world)
    klo, khi = kx_r[rank]
    nk = khi - klo
    dtype = torch.complex128 if precision == 64 else torch.complex64
    dev = f"cuda:{_lib.ensure_device()}"
    st = torch.cuda.current_stream().cuda_stream
    c = g.center()
    s = np.ascontiguousarray(R @ c - c + np.asarray(g.origin), dtype=np.float64)
    dom = np.ascontiguousarray(g.delta_omega(), dtype=np.float64)
    q = torch.empty((nk, w[1], w[2]), dtype=dtype, device=dev)
    _lib.check(_lib.LIB.gf_rotate_product_planes(C1.handle, C2.handle, int(bool(wrap)), _lib.dptr(dom),
                                                 _lib.dptr(np.ascontiguousarray(R)), _lib.dptr(s), precision, klo, nk,
                                                 ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(st)))
    a = _pass(q, (nk, w[1], N[2]), 2, N[2], 1.0, precision)
    ny = y_r[rank][1] - y_r[rank][0]
    if exchange == "auto":
        dist = _dist()
        exchange = "fused" if dist.is_initialized() and dist.get_backend(group) == "nccl" else "alltoall"
    if exchange == "fused":
        ny_max = max(hi - lo for lo, hi in y_r)
        buf, hdl = _symm_slab((w[0], ny_max, N[2]), dtype, group)
        hdl.barrier()  # every rank is done with its slab from the previous call
        bounds = [lo for lo, _ in y_r] + [y_r[-1][1]]
        scatter_y_pass(a.contiguous(), N[1], bounds, list(hdl.buffer_ptrs), klo, precision)
        hdl.barrier()  # every rank's stores into this slab have landed
        slab = torch.view_as_complex(buf.view(-1)[: 2 * w[0] * ny * N[2]].view(w[0], ny, N[2], 2))
    else:
        b = _pass(a, (nk, N[1], N[2]), 1, N[1], 1.0, precision)
        slab = exchange_planes_to_slabs(torch.view_as_real(b), kx_r, y_r, rank, group)
        slab = torch.view_as_complex(slab.contiguous())
    scale = 1.0 / (g.node_count * g.cell_volume)
    return _pass(slab, (N[0], ny, N[2]), 0, N[0], scale, precision)


def _pass(x, out_shape, axis, n, scale, precision):
    import torch

    out = torch.empty(out_shape, dtype=x.dtype, device=x.device)
    if x.numel() == 0 or out.numel() == 0:
        return out
    si = (ctypes.c_int32 * 3)(*x.shape)
    so = (ctypes.c_int32 * 3)(*out_shape)
    st = torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.LIB.gf_fft_pass(precision, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), si, so,
                                    axis, n, 1, 0, 1, 0.0, 0.0, float(scale), ctypes.c_void_p(st)))
    return out


# ---------------------------------------------------------------------------
# density node slabs


def density_slab_plan(n0, world):
    """Per rank: (plane0, nplanes, halo_lo, halo_hi) over axis 0."""
    plan = []
    for r in range(world):
        lo, hi = shard_range(n0, r, world)
        plan.append((lo, hi - lo, 1 if 0 < lo < hi else 0, 1 if lo < hi < n0 else 0))
    return plan


def affinity_field_slab(solid, grid, spec, policy=None, group=None, gather=True, compute=None):
    """affinity_field with the grid's axis-0 planes sharded across ranks.

    Each rank runs the GPU pipeline on its slab (gf_affinity_planes: global
    node indexing, halo planes for the neighbour fill), so every node's
    value and flag is bit-identical to the single-GPU affinity_field.
    gather=True returns the full ComplexField on every rank; otherwise
    (local values (nplanes * plane,), plane range, local flags, stats).
    `compute(solid, grid, plane0, nplanes, halo_lo, halo_hi)` may replace
    the GPU call (tests drive the decomposition on CPU)."""
    import torch

    from .descriptor import ComplexField, IntegrationPolicy, _check_grid, _unit_constant

    policy = policy or IntegrationPolicy()
    _check_grid(solid, grid)
    rank, world = _world(group)
    plane0, n, hlo, hhi = density_slab_plan(grid.dims[0], world)[rank]
    plane = int(np.prod(grid.dims[1:]))
    family = 0 if spec.family == "InverseSquare" else 1
    if compute is None:
        def compute(solid, grid, p0, np_, lo, hi):
            return backend.affinity_planes(solid, grid, p0, np_, lo, hi, family, spec.sigma,
                                           _unit_constant(grid.dimension), spec.lambda_in, spec.lambda_out,
                                           policy.max_solid_angle, policy.max_recursion_depth, policy.eta_floor)
    if n > 0:
        values, fb, st = compute(solid, grid, plane0, n, hlo, hhi)
        nclamp, worst = st[0], st[1]
    else:
        values = torch.empty(0, dtype=torch.complex128)
        fb = torch.empty(0, dtype=torch.uint8)
        nclamp, worst = 0, 0.0
    fb_h = fb.cpu().numpy()
    excluded, unresolved, inside = (fb_h & 1) != 0, (fb_h & 2) != 0, (fb_h & 4) != 0
    local_flags = (np.flatnonzero(excluded | unresolved) + plane0 * plane).tolist()
    counts = torch.tensor([int(excluded.sum()), int(unresolved.sum()), int(inside.sum()), int(nclamp)],
                          dtype=torch.float64)
    worst_t = torch.tensor([float(worst)], dtype=torch.float64)
    flags = local_flags
    if world > 1:
        dist = _dist()
        dev = values.device if values.is_cuda else torch.device("cpu")
        if dist.get_backend(group) == "nccl":
            counts, worst_t = counts.to(dev), worst_t.to(dev)
        dist.all_reduce(counts, group=group)
        dist.all_reduce(worst_t, op=dist.ReduceOp.MAX, group=group)
        if gather:
            parts = [None] * world
            dist.all_gather_object(parts, local_flags, group=group)
            flags = [f for p in parts for f in p]  # ranks own increasing plane ranges: already sorted
    c = counts.cpu().numpy()
    stats = {"excluded": int(c[0]), "eta_clamped": int(c[3]),
             "worst_residual": float(worst_t.cpu()[0]) if family else 0.0,
             "unresolved_nodes": int(c[1]), "inside_nodes": int(c[2])}
    if not gather:
        return values, (plane0, plane0 + n), local_flags, stats
    full = gather_rows(values.reshape(n, plane), grid.dims[0], group).reshape(-1)
    return ComplexField(grid, full, flags=flags, stats=stats)


# ---------------------------------------------------------------------------
# forward window of a node-sharded field


def _wpass(x, out_shape, axis, n, scale, precision):
    """One pruned forward pass: node-ordered in, DC-centred window out with
    the (-1)^m centre phase (spectral.forward_window's per-axis pass)."""
    import torch

    out = torch.empty(out_shape, dtype=x.dtype, device=x.device)
    if x.numel() == 0 or out.numel() == 0:
        return out
    si = (ctypes.c_int32 * 3)(*x.shape)
    so = (ctypes.c_int32 * 3)(*out_shape)
    st = torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.LIB.gf_fft_pass(precision, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), si, so,
                                    axis, n, 0, 1, -1, 0.0, 0.5, float(scale), ctypes.c_void_p(st)))
    return out


def window_inner_passes(local, dims, w, precision=64):
    """z then y pass of a rank's (nx, N1, N2) field planes -> (nx, w, w)."""
    nx = local.shape[0]
    a = _wpass(local, (nx, dims[1], w), 2, dims[2], 1.0, precision)
    return _wpass(a, (nx, w, w), 1, dims[1], 1.0, precision)


def window_outer_pass(slab, dims, w, cell_volume, precision=64):
    """x pass of a (N0, wy, w) window y-slab -> (w, wy, w), scaled by dV."""
    return _wpass(slab, (w, slab.shape[1], w), 0, dims[0], cell_volume, precision)


def forward_window_slab(local, grid, w, precision=64, group=None, gather=True, exchange="auto"):
    """spectral.forward_window for a field sharded by axis-0 planes
    (shard_range layout, local = this rank's (nx, N1, N2) CUDA complex
    planes).  Bit-identical to the single-GPU window: the same 1-D passes on
    the same data, with one all-to-all between the y and x passes.  Returns
    the full (w, w, w) window on every rank (gather) or this rank's window
    y-slab (w, wy, w) and its range."""
    import torch

    if grid.dimension != 3:
        raise ValueError("slab decomposition is for 3D fields")
    rank, world = _world(group)
    N = list(grid.dims)
    dtype = torch.complex128 if precision == 64 else torch.complex64
    local = local.reshape(-1, N[1], N[2]).to(dtype)
    x_r = [shard_range(N[0], r, world) for r in range(world)]
    wy_r = [shard_range(w, r, world) for r in range(world)]
    if exchange == "auto":
        dist = _dist()
        exchange = "fused" if dist.is_initialized() and dist.get_backend(group) == "nccl" else "alltoall"
    if exchange == "fused":  # y pass stores straight into the peers' window y-slabs
        nx = local.shape[0]
        a = _wpass(local, (nx, N[1], w), 2, N[2], 1.0, precision)
        wy_max = max(hi - lo for lo, hi in wy_r)
        buf, hdl = _symm_slab((N[0], wy_max, w), dtype, group)
        hdl.barrier()
        bounds = [lo for lo, _ in wy_r] + [wy_r[-1][1]]
        scatter_y_pass(a.contiguous(), N[1], bounds, list(hdl.buffer_ptrs), x_r[rank][0], precision, forward=True)
        hdl.barrier()
        wy = wy_r[rank][1] - wy_r[rank][0]
        slab = torch.view_as_complex(buf.view(-1)[: 2 * N[0] * wy * w].view(N[0], wy, w, 2))
    else:
        b = window_inner_passes(local, N, w, precision)
        slab = exchange_planes_to_slabs(torch.view_as_real(b), x_r, wy_r, rank, group)
        slab = torch.view_as_complex(slab.contiguous())
    out = window_outer_pass(slab, N, w, grid.cell_volume, precision)
    if not gather:
        return out, wy_r[rank]
    full = gather_rows(torch.view_as_real(out.permute(1, 0, 2).contiguous()), w, group)
    return torch.view_as_complex(full.contiguous()).permute(1, 0, 2).contiguous()
