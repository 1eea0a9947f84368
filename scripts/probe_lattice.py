"""Lattice-aligned poses (identity, screws about a grid axis) put every mode
on an integer reference index; compare their cost with generic rotations for
the batched sweep (w=96) and the 512^3 landscape."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be, _lib
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.energy import score_field_device
from conftest import synthetic_window, random_rotation
_lib.ensure_device(0)
rng = np.random.default_rng(0)


def timeit(f, n=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(n):
        e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best


def zrot(a):
    c, s = np.cos(a), np.sin(a)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


w = 96
W1, W2 = be.DeviceWindow(synthetic_window(rng, w)), be.DeviceWindow(synthetic_window(rng, w))
n = 4096
sets = {"random": np.stack([random_rotation(rng) for _ in range(n)]),
        "z-screw": np.stack([zrot(a) for a in rng.uniform(0, 2 * np.pi, n)]),
        "identity": np.stack([np.eye(3)] * n)}
ts = rng.uniform(-0.5, 0.5, (n, 3))
for name, Rs in sets.items():
    poses = torch.from_numpy(be.pack_poses(Rs, ts)).cuda()
    out = torch.empty((n, 14), dtype=torch.float64, device="cuda")
    ms = timeit(lambda: be.cascade_batch(W1, W2, False, (1.0 / (2 * w * 0.05),) * 3, 1.0, [0.1, 0.2, 0.3], poses,
                                         out=out, precision="fp32"))
    print(f"sweep w={w} {name:9s}: {n / ms * 1e3:9.0f} poses/s", flush=True)
del W1, W2
N = 512
g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
torch.manual_seed(0)
C1 = be.DeviceWindow(torch.randn((N,) * 3, dtype=torch.complex128, device="cuda"))
C2 = be.DeviceWindow(torch.randn((N,) * 3, dtype=torch.complex128, device="cuda"))


class A:
    def __init__(s, win): s.grid, s.w = g, win
    def window(s, m=None): return s.w, True


for name, R in (("random", random_rotation(rng)), ("z-screw", zrot(0.7)), ("identity", np.eye(3))):
    ms = timeit(lambda: score_field_device(A(C1), A(C2), R, None, precision=32))
    print(f"landscape 512^3 {name:9s}: {ms:.3f} ms", flush=True)
