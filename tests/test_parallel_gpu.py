"""Single-rank GPU runs of the multi-GPU paths (the decomposition itself is
tested at world size 2 with gloo in test_parallel.py)."""

import numpy as np
import pytest

import oracle
from paper_1711_05017_b200 import parallel
from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid
from paper_1711_05017_b200.energy import Configuration, PartAsset, evaluate, score_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def assets():
    rng = np.random.default_rng(4)
    g = SampleGrid(3, (32, 32, 32), (-1.6, -1.6, -1.6), 0.1)
    mk = lambda: ComplexField(g, rng.normal(size=g.node_count) + 1j * rng.normal(size=g.node_count))  # noqa: E731
    return PartAsset.from_field("a", mk()), PartAsset.from_field("b", mk(), movable=True)


def test_pose_sweep_matches_evaluate(assets):
    a1, a2 = assets
    Rs, ts = oracle.bench_poses(40, 0.5, seed=1)
    for prec, tol in (("fp64", 1e-10), ("fp32", 1e-4)):
        out = parallel.pose_sweep(a1, a2, Rs, ts, m_prime=16 ** 3, precision=prec)
        assert out.shape == (40, 7)
        from paper_1711_05017_b200 import backend

        backend.set_precision(prec)
        try:
            for i in range(0, 40, 7):
                ev = evaluate(a1, a2, Configuration(Rs[i], ts[i]), 16 ** 3)
                assert abs(out[i, 0] - ev.score) <= tol * max(abs(ev.score), 1e-3)
                np.testing.assert_allclose(out[i, 1:4].real, ev.force, rtol=tol, atol=tol * np.max(np.abs(ev.force)))
        finally:
            backend.set_precision("fp32")


@pytest.mark.parametrize("mp", [16 ** 3, None])
def test_score_field_slab_equals_score_field(assets, mp):
    a1, a2 = assets
    R = oracle.quat_rotation([0.7, -0.3, 0.2, 0.4])
    full = score_field(a1, a2, R, mp).values.reshape(32, 32, 32)
    slab = parallel.score_field_slab(a1, a2, R, mp).cpu().numpy()
    np.testing.assert_allclose(slab, full, atol=1e-11 * np.max(np.abs(full)))


@pytest.mark.parametrize("world,mp,prec", [(2, None, 64), (3, 16 ** 3, 64), (4, None, 32)])
def test_fused_scatter_exchange_simulated_ranks(assets, world, mp, prec):
    """The fused y pass + exchange (gf_fft_pass_scatter) for `world` ranks,
    simulated on one GPU: every rank's pass writes straight into all ranks'
    slab buffers (no rank waits on another), then each slab gets its x pass.
    The slabs reassemble -- bit for bit -- into the single-GPU landscape."""
    import ctypes

    import torch

    from paper_1711_05017_b200 import _lib
    from paper_1711_05017_b200.energy import score_field_device

    a1, a2 = assets
    R = oracle.quat_rotation([0.7, -0.3, 0.2, 0.4])
    g = a1.grid
    N = list(g.dims)
    C1, wrap1 = a1.window(mp)
    C2, wrap2 = a2.window(mp)
    w = list(C1.shape)
    want = score_field_device(a1, a2, R, mp, precision=prec).reshape(N)
    dtype = torch.complex128 if prec == 64 else torch.complex64
    kx_r, y_r = parallel.slab_plan(w, N, world)
    slabs = [torch.zeros((w[0], hi - lo, N[2]), dtype=dtype, device="cuda") for lo, hi in y_r]
    bounds = [lo for lo, _ in y_r] + [y_r[-1][1]]
    c = g.center()
    s = np.ascontiguousarray(R @ c - c + np.asarray(g.origin), dtype=np.float64)
    dom = np.ascontiguousarray(g.delta_omega(), dtype=np.float64)
    st = torch.cuda.current_stream().cuda_stream
    for klo, khi in kx_r:
        q = torch.empty((khi - klo, w[1], w[2]), dtype=dtype, device="cuda")
        _lib.check(_lib.LIB.gf_rotate_product_planes(C1.handle, C2.handle, int(wrap1 and wrap2), _lib.dptr(dom),
                                                     _lib.dptr(np.ascontiguousarray(R)), _lib.dptr(s), prec, klo,
                                                     khi - klo, ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(st)))
        a = parallel._pass(q, (khi - klo, w[1], N[2]), 2, N[2], 1.0, prec)
        parallel.scatter_y_pass(a, N[1], bounds, [t.data_ptr() for t in slabs], klo, prec)
    scale = 1.0 / (g.node_count * g.cell_volume)
    got = torch.cat([parallel._pass(sl, (N[0], sl.shape[1], N[2]), 0, N[0], scale, prec) for sl in slabs], dim=1)
    assert torch.equal(got, want)


def test_fused_exchange_through_symmetric_memory_single_rank(assets):
    """score_field_slab(exchange="fused") through a real NCCL process group and
    symmetric-memory rendezvous (world size 1 on this box) equals the
    all-to-all path."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    a1, a2 = assets
    R = oracle.quat_rotation([0.2, 0.5, -0.6, 0.1])
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        fused = parallel.score_field_slab(a1, a2, R, None, exchange="fused")
        plain = parallel.score_field_slab(a1, a2, R, None, exchange="alltoall")
        assert torch.equal(fused, plain)
        g = a1.grid
        x = torch.randn(g.dims, dtype=torch.complex128, device="cuda")
        wf = parallel.forward_window_slab(x, g, 16, exchange="fused")
        wa = parallel.forward_window_slab(x, g, 16, exchange="alltoall")
        assert torch.equal(wf, wa)
    finally:
        parallel._SYMM.clear()
        dist.destroy_process_group()
