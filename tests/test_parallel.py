"""Multi-rank decomposition logic on CPU (gloo, world size 2).

The pose sweep's sharding + gather and the landscape's plane -> slab
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
from paper_1711_05017_b200 import parallel


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
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sweep_and_slab_decomposition_gloo(world):
    manager = mp.Manager()
    results = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        assert results[f"sweep{r}"] <= 1e-12
        assert results[f"field{r}"] <= 1e-12


def test_shard_range_partitions():
    for n in (0, 1, 7, 100, 1000003):
        for world in (1, 2, 3, 8):
            parts = [parallel.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
