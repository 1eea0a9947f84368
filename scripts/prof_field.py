"""ncu workload: one 512^3 full-spectrum fp32 landscape (after a warm-up)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1711_05017_b200 import backend, _lib
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.energy import score_field_device
_lib.ensure_device(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = int(sys.argv[2]) if len(sys.argv) > 2 else N
g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
C1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda"))
C2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda"))
class A:
    def __init__(s, win): s.grid, s.w = g, win
    def window(s, m=None): return s.w, w == N
R = np.array([[0.36, 0.48, -0.8], [-0.8, 0.6, 0.0], [0.48, 0.64, 0.6]])
for _ in range(3):
    out = score_field_device(A(C1), A(C2), R, None, precision=32)
torch.cuda.synchronize()
print("done", out.shape)
