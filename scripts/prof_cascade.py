"""Small fixed workload for ncu: single-query (serial) and batched cascade at w=64."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be
from conftest import synthetic_window, random_rotation

mode = sys.argv[1] if len(sys.argv) > 1 else "batch"
w = int(sys.argv[2]) if len(sys.argv) > 2 else 64
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
rng = np.random.default_rng(0)
from paper_1711_05017_b200 import _lib
_lib.ensure_device(0)
C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
dom = (1.0 / (2 * w * 0.05),) * 3
n = 2048 if mode == "batch" else 8
Rs = np.stack([random_rotation(rng) for _ in range(n)]); tt = rng.uniform(-1, 1, (n, 3))
poses = torch.from_numpy(be.pack_poses(Rs, tt)).cuda()
out = torch.empty((n, 14), dtype=torch.float64, device="cuda")
for _ in range(3):
    be.cascade_batch(W1, W2, False, dom, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision=prec, serial=(mode != "batch"))
torch.cuda.synchronize()
print("done")
