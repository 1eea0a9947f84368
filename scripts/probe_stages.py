"""GPU probe: timings of stages W (forward window), F (landscape), D (density), Q3 (sweep)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1711_05017_b200 import backend, scenes, parallel, _lib
from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid, KernelSpec, affinity_field
from paper_1711_05017_b200.energy import PartAsset, score_field_device
from paper_1711_05017_b200.spectral import forward_window, Spectrum

_lib.ensure_device(0)


def _rand_rot(seed=1):
    q = np.random.default_rng(seed).normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
dev = "cuda:0"
which = sys.argv[1:] or ["W", "F", "D", "S"]

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

class FakeAsset:
    def __init__(self, grid, win, wrap):
        self.grid, self._w, self._wrap = grid, win, wrap
    def window(self, m_prime=None):
        return self._w, self._wrap

if "W" in which:
    for N, w in ((256, 96), (512, 128), (256, 256)):
        g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
        x = torch.randn(N ** 3, dtype=torch.complex128, device=dev)
        f = ComplexField(g, x)
        ms = timeit(lambda: forward_window(f, w))
        byt = 16 * N ** 3 + 16 * w ** 3
        print(f"W forward_window N={N} w={w} complex128: {ms:.3f} ms  {byt / ms / 1e6:.0f} GB/s (alg bytes)", flush=True)

if "F" in which:
    for N, w, prec in ((256, 256, 32), (512, 512, 32), (512, 128, 32), (256, 256, 64)):
        g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
        C1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device=dev))
        C2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device=dev))
        a1, a2 = FakeAsset(g, C1, w == N), FakeAsset(g, C2, w == N)
        R = _rand_rot()
        ms = timeit(lambda: score_field_device(a1, a2, R, None, precision=prec))
        eb = 8 if prec == 32 else 16
        byt = 2 * eb * w ** 3 + eb * N ** 3
        print(f"F score_field N={N} w={w} fp{prec}: {ms:.3f} ms  {N**3 / ms / 1e6:.1f} Gvox/s  {byt / ms / 1e6:.0f} GB/s alg", flush=True)
        del C1, C2
        torch.cuda.empty_cache()

if "D" in which:
    for name, n in (("peg_in_hole", 64), ("peg_in_hole", 128), ("gear_pair", 128)):
        sc = scenes.get_scene(name)
        g = sc.grid(n)
        for solid in (sc.fixed,):
            t0 = time.perf_counter()
            f = affinity_field(solid, g, sc.kernel)
            dt = time.perf_counter() - t0
            t0 = time.perf_counter()
            f = affinity_field(solid, g, sc.kernel)
            dt = time.perf_counter() - t0
            nf = len(solid.mesh.faces)
            print(f"D affinity {name} n={n} faces={nf}: {dt*1e3:.1f} ms  {g.node_count/dt/1e6:.2f} Mvox/s  "
                  f"{g.node_count*nf/dt/1e9:.2f} Gpairs/s  excluded={f.stats['excluded']} unresolved={f.stats['unresolved_nodes']}", flush=True)

if "S" in which:
    for w in (64, 96):
        g = SampleGrid(3, (256,) * 3, (-2.7,) * 3, 5.42 / 256)
        C1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device=dev) * 0.01)
        C2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device=dev) * 0.01)
        a1, a2 = FakeAsset(g, C1, False), FakeAsset(g, C2, False)
        import oracle
        Rs, ts = oracle.bench_poses(8192, 0.25 * 5.42, seed=0)
        parallel.pose_sweep(a1, a2, Rs[:64], ts[:64], precision="fp32")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        parallel.pose_sweep(a1, a2, Rs, ts, precision="fp32")
        dt = time.perf_counter() - t0
        print(f"S pose_sweep w={w}: {len(ts)/dt:.0f} poses/s (incl. host pose packing + D2H)", flush=True)
