"""Lone-query kernel vs the batched kernel on one or two poses at large windows."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be, _lib
from conftest import synthetic_window, random_rotation
_lib.ensure_device(0)
rng = np.random.default_rng(0)
for w in (64, 96, 128):
    W1, W2 = be.DeviceWindow(synthetic_window(rng, w)), be.DeviceWindow(synthetic_window(rng, w))
    n = 64
    Rs = np.stack([random_rotation(rng) for _ in range(n)]); ts = rng.uniform(-1, 1, (n, 3))
    poses = torch.from_numpy(be.pack_poses(Rs, ts)).cuda()
    out = torch.empty((n, 14), dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for serial in (True, False):
        be.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses, out=out, serial=serial)
        torch.cuda.synchronize(); e0.record()
        be.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses, out=out, serial=serial)
        e1.record(); torch.cuda.synchronize()
        print(f"w={w} {'serial lone-query kernel' if serial else 'batched kernel (64 poses)'}: {e0.elapsed_time(e1) * 1e3 / n:.2f} us/pose")
    for k in (2, 4, 8):
        be.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses[:k], out=out[:k])
        torch.cuda.synchronize(); e0.record()
        for _ in range(10):
            be.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses[:k], out=out[:k])
        e1.record(); torch.cuda.synchronize()
        print(f"w={w} batched kernel, {k} poses per launch: {e0.elapsed_time(e1) * 1e3 / 10:.2f} us/launch")
