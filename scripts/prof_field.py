"""ncu workload: one 512^3 full-spectrum fp32 landscape (after a warm-up)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1711_05017_b200 import backend, _lib
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.energy import score_field_device
_lib.ensure_device(0)


def _rand_rot(seed=1):
    q = np.random.default_rng(seed).normal(size=4)
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = int(sys.argv[2]) if len(sys.argv) > 2 else N
g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
C1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda"))
C2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda"))
class A:
    def __init__(s, win): s.grid, s.w = g, win
    def window(s, m=None): return s.w, w == N
R = _rand_rot()
for _ in range(3):
    out = score_field_device(A(C1), A(C2), R, None, precision=32)
torch.cuda.synchronize()
print("done", out.shape)
