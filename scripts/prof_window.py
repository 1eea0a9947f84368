"""ncu workload: forward centred window 256^3 complex128 -> 96^3 (bench stage W)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1711_05017_b200 import _lib
from paper_1711_05017_b200.descriptor import ComplexField, SampleGrid
from paper_1711_05017_b200.spectral import forward_window
_lib.ensure_device(0)
N, w = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (256, 96)
g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
f = ComplexField(g, torch.randn(N ** 3, dtype=torch.complex128, device="cuda"))
for _ in range(3):
    out = forward_window(f, w)
torch.cuda.synchronize()
print("done", out.shape)
