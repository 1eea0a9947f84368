"""C3-style sweep timing: w=96 fp32, cmd_bench poses, one batched launch."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle
from paper_1711_05017_b200 import backend as be, _lib
from conftest import synthetic_window
_lib.ensure_device(0)
if os.environ.get('GF_RUNLEN'):
    _lib.check(_lib.LIB.gf_set_cascade_run_length(int(os.environ['GF_RUNLEN'])))
rng = np.random.default_rng(0)
w = int(sys.argv[1]) if len(sys.argv) > 1 else 96
W1, W2 = be.DeviceWindow(synthetic_window(rng, w)), be.DeviceWindow(synthetic_window(rng, w))
Rs, ts = oracle.bench_poses(8192, 0.5, seed=0)
poses = torch.from_numpy(be.pack_poses(Rs, ts)).cuda()
out = torch.empty((len(ts), 14), dtype=torch.float64, device="cuda")
f = lambda: be.cascade_batch(W1, W2, False, (1.0 / (2 * w * 0.05),) * 3, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision="fp32")
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(); f(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(f"w={w} {len(ts)} poses: {best:.2f} ms  {len(ts) / best * 1e3:.0f} poses/s")
