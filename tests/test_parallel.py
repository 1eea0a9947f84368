"""Multi-rank decomposition logic on CPU (gloo, world size 2).

The pose sweep's sharding + gather, the landscape's plane -> slab
all-to-all and the node-sharded forward window's plane -> window-slab
all-to-all run through the same host code the GPU path uses; the per-rank
compute is the oracle (numpy / C restatement), so the test checks the
decomposition, not the kernels (those are covered by the -m gpu suite).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1711_05017_b200 import parallel, scenes
from paper_1711_05017_b200.descriptor import KernelSpec, SampleGrid


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _windows(w=8, seed=0):
    rng = np.random.default_rng(seed)
    k = np.stack(np.meshgrid(*[np.arange(w) - w // 2] * 3, indexing="ij"), axis=-1)
    amp = 1.0 / (1.0 + np.sum(k * k, axis=-1))
    mk = lambda: (rng.normal(size=(w,) * 3) + 1j * rng.normal(size=(w,) * 3)) * amp  # noqa: E731
    return mk(), mk()


DOM = (0.2, 0.2, 0.2)
CEN = np.array([0.1, -0.2, 0.3])


def _oracle_compute(C1, C2):
    def compute(_a1, _a2, Rs, ts):
        rows = [oracle.cascade(C1, C2, False, DOM, 0.5, R, t - CEN + R @ CEN, CEN) for R, t in zip(Rs, ts)]
        return np.asarray(rows).reshape(len(ts), 7)

    return compute


def _centred_inverse(x, axis, n):
    """numpy: window-centred input along axis -> n node outputs, unnormalised."""
    w = x.shape[axis]
    shape = list(x.shape)
    shape[axis] = n
    full = np.zeros(shape, dtype=np.complex128)
    idx = [slice(None)] * x.ndim
    for k in range(w):
        idx[axis] = (k - w // 2) % n
        src = [slice(None)] * x.ndim
        src[axis] = k
        full[tuple(idx)] = x[tuple(src)]
    return np.fft.ifft(full, axis=axis) * n


def _centred_forward(x, axis, w):
    """numpy: node-ordered input along axis -> the DC-centred w-mode window
    of fftshift(fft(ifftshift(x))) (one pruned forward pass)."""
    n = x.shape[axis]
    y = np.fft.fftshift(np.fft.fft(np.fft.ifftshift(x, axes=axis), axis=axis), axes=axis)
    return np.take(y, np.arange(n // 2 - w // 2, n // 2 + w // 2), axis=axis)


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        C1, C2 = _windows()
        # --- pose sweep: sharded + gathered == serial
        Rs, ts = oracle.bench_poses(9, 0.5, seed=0)
        got = parallel.pose_sweep(None, None, Rs, ts, compute=_oracle_compute(C1, C2))
        want = _oracle_compute(C1, C2)(None, None, Rs, ts)
        results[f"sweep{rank}"] = float(np.max(np.abs(got - want)))
        # --- landscape: planes -> slabs exchange
        N = (16, 16, 16)
        h = 0.1
        origin = tuple(-0.8 for _ in N)
        R = oracle.quat_rotation([0.9, 0.2, -0.1, 0.3])
        w = C1.shape
        kx_r, y_r = parallel.slab_plan(w, N, world)
        klo, khi = kx_r[rank]
        c = oracle.grid_center(N, origin, h)
        dom = np.array([1.0 / (n * h) for n in N])
        W = oracle.window_freqs(w, dom)
        u = -(W @ R) / dom + np.asarray([x // 2 for x in w])
        V, _ = oracle.interp_window(C2, u, False)
        s = R @ c - c + np.asarray(origin)
        Q = (C1.ravel() * V * np.exp(2j * np.pi * (W @ s))).reshape(w)[klo:khi]
        a = _centred_inverse(Q, 2, N[2])
        b = _centred_inverse(a, 1, N[1])
        slab = parallel.exchange_planes_to_slabs(torch.view_as_real(torch.from_numpy(b)), kx_r, y_r, rank)
        slab = torch.view_as_complex(slab.contiguous()).numpy()
        land = _centred_inverse(slab, 0, N[0]) / (np.prod(N) * h ** 3)
        full = oracle.score_field(C1, C2, False, N, origin, h, R)
        ylo, yhi = y_r[rank]
        results[f"field{rank}"] = float(np.max(np.abs(land - full[:, ylo:yhi])) / np.max(np.abs(full)))
        # --- forward window of a node-sharded field: z, y passes on the
        # rank's planes -> all-to-all -> x pass (parallel.forward_window_slab's plan)
        rng = np.random.default_rng(7)
        f = rng.normal(size=N) + 1j * rng.normal(size=N)
        wn = 8
        x_r = [parallel.shard_range(N[0], r, world) for r in range(world)]
        wy_r = [parallel.shard_range(wn, r, world) for r in range(world)]
        xlo, xhi = x_r[rank]
        pz = _centred_forward(f[xlo:xhi], 2, wn)
        py = _centred_forward(pz, 1, wn)
        slab = parallel.exchange_planes_to_slabs(torch.view_as_real(torch.from_numpy(py)), x_r, wy_r, rank)
        slab = torch.view_as_complex(slab.contiguous()).numpy()
        win = _centred_forward(slab, 0, wn) * h ** 3
        want = oracle.center_window(oracle.forward_dft(f, N, origin, h), N, origin, h, wn)
        wlo, whi = wy_r[rank]
        results[f"window{rank}"] = float(np.max(np.abs(win - want[:, wlo:whi])) / np.max(np.abs(want)))
        # --- density node slabs: halo planes make the neighbour fill exact
        g = SampleGrid(3, (8, 8, 8), (-0.8, -0.8, -0.8), 0.2)
        solid = scenes.box_mesh((0.2, 0.2, 0.2))
        got = parallel.affinity_field_slab(solid, g, KernelSpec(), compute=_fake_planes)
        want_v, want_fb, (want_cl, want_w) = _fake_planes(solid, g, 0, g.dims[0], 0, 0)
        wfb = want_fb.numpy()
        ok = (np.array_equal(got.values, want_v.numpy()) and
              got.flags == np.flatnonzero((wfb & 3) != 0).tolist() and
              got.stats["excluded"] == int(((wfb & 1) != 0).sum()) and
              got.stats["inside_nodes"] == int(((wfb & 4) != 0).sum()) and
              got.stats["eta_clamped"] == want_cl and got.stats["worst_residual"] == want_w)
        results[f"density{rank}"] = bool(ok)
    finally:
        dist.destroy_process_group()


def _fake_planes(solid, grid, p0, n, lo, hi):
    """Deterministic stand-in for gf_affinity_planes: per-node values from
    global coordinates, an excluded set, and the neighbour fill over the
    computed block (owned + halo planes), returning the owned planes."""
    a, b = p0 - lo, p0 + n + hi
    idx = np.stack(np.meshgrid(np.arange(a, b), *[np.arange(m) for m in grid.dims[1:]], indexing="ij"), -1)
    x = np.asarray(grid.origin) + grid.spacing * idx
    raw = np.sin(3 * x[..., 0]) + 1j * np.cos(x[..., 1] * x[..., 2] + x[..., 0])
    ex = raw.real > 0.6
    unres = (idx.sum(-1) % 5) == 0
    inside = raw.imag > 0.5
    dims = (b - a,) + tuple(grid.dims[1:])
    vals = oracle.neighbor_average(raw.ravel(), ex.ravel(), dims).reshape(dims)
    fb = (ex.astype(np.uint8) | (unres.astype(np.uint8) << 1) | (inside.astype(np.uint8) << 2))
    own = slice(lo, lo + n)
    resid = np.abs(raw[own]).ravel()
    return (torch.from_numpy(vals[own].ravel().copy()), torch.from_numpy(fb[own].ravel().copy()),
            (int(unres[own].sum()), float(resid.max())))


@pytest.mark.parametrize("world", [2])
def test_sweep_and_slab_decomposition_gloo(world):
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        assert results[f"sweep{r}"] <= 1e-12
        assert results[f"field{r}"] <= 1e-12
        assert results[f"window{r}"] <= 1e-12
        assert results[f"density{r}"]


def test_density_slab_plan():
    for n0 in (4, 8, 9, 64):
        for world in (1, 2, 3, 8):
            plan = parallel.density_slab_plan(n0, world)
            assert sum(p[1] for p in plan) == n0
            for p0, n, lo, hi in plan:
                assert p0 - lo >= 0 and p0 + n + hi <= n0
                if n:
                    assert lo == (1 if p0 > 0 else 0) and hi == (1 if p0 + n < n0 else 0)


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 1000003):
        for world in (1, 2, 3, 8):
            parts = [parallel.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
