"""Time the fp32 landscape score_field_device at N^3 (argv: N, w, reps)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_05017_b200 import _lib, backend  # noqa: E402
from paper_1711_05017_b200.descriptor import SampleGrid  # noqa: E402
from paper_1711_05017_b200.energy import score_field_device  # noqa: E402

_lib.ensure_device(0)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
w = int(sys.argv[2]) if len(sys.argv) > 2 else N
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
g = SampleGrid(3, (N,) * 3, (-1.0,) * 3, 2.0 / N)
W1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda"))
W2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda"))


class A:
    def __init__(s, win):
        s.grid, s.w = g, win

    def window(s, m=None):
        return s.w, w == N


rng = np.random.default_rng(1)
for name, R in (("random", None), ("identity", np.eye(3))):
    if R is None:
        q = rng.normal(size=4)
        q /= np.linalg.norm(q)
        ww, x, y, z = q
        R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - ww * z), 2 * (x * z + ww * y)],
                      [2 * (x * y + ww * z), 1 - 2 * (x * x + z * z), 2 * (y * z - ww * x)],
                      [2 * (x * z - ww * y), 2 * (y * z + ww * x), 1 - 2 * (x * x + y * y)]])
    for _ in range(2):
        score_field_device(A(W1), A(W2), R, None, precision=32)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        score_field_device(A(W1), A(W2), R, None, precision=32)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{name}: N={N} w={w} best {ms:.3f} ms median {sorted(ts)[len(ts)//2]:.3f} ms "
          f"frac(24B/vox) {24 * N**3 / (ms * 1e-3) / 1e9 / 6549.1:.3f}", flush=True)
