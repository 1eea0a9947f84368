"""Quick GPU probe: cascade single-query latency and batch throughput."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import synthetic_window, random_rotation

rng = np.random.default_rng(0)
import ctypes
from paper_1711_05017_b200 import _lib
_lib.ensure_device(0)
L = int(os.environ.get('RUNLEN', '0'))
_lib.check(_lib.LIB.gf_set_cascade_run_length(L))
VAR = int(os.environ.get('VARIANT', '1'))
_lib.check(_lib.LIB.gf_set_cascade_variant(VAR))
_lib.check(_lib.LIB.gf_set_cascade_tile(int(os.environ.get('TILE','0'))))
WS = [int(x) for x in os.environ.get('WS', '32,64,96,128').split(',')]
PRECS = os.environ.get('PRECS', 'fp32,fp64').split(',')
torch.cuda.init()
print(torch.cuda.get_device_name(), flush=True)
for prec in PRECS:
    for w in WS:
        C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
        W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
        dom = (1.0 / (2 * w * 0.05),) * 3
        # single query host in/out
        ts = []
        for i in range(300):
            R = random_rotation(rng); t = rng.uniform(-1, 1, 3)
            t0 = time.perf_counter_ns()
            be.cascade(W1, W2, False, dom, 1.0, R, t, [0.1, 0.2, 0.3], precision=prec)
            ts.append((time.perf_counter_ns() - t0) / 1e3)
        ts = sorted(ts[20:])
        p50 = ts[len(ts) // 2]; p99 = ts[min(len(ts) - 1, int(0.99 * len(ts)))]
        # serial device loop
        n = 200
        Rs = np.stack([random_rotation(rng) for _ in range(n)]); tt = rng.uniform(-1, 1, (n, 3))
        poses = torch.from_numpy(be.pack_poses(Rs, tt)).cuda()
        out = torch.empty((n, 14), dtype=torch.float64, device="cuda")
        be.cascade_batch(W1, W2, False, dom, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision=prec, serial=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        be.cascade_batch(W1, W2, False, dom, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision=prec, serial=True)
        e1.record(); torch.cuda.synchronize()
        ser_us = e0.elapsed_time(e1) * 1e3 / n
        # batch throughput
        nb = 4096 if w <= 64 else 1024
        Rs = np.stack([random_rotation(rng) for _ in range(nb)]); tt = rng.uniform(-1, 1, (nb, 3))
        poses = torch.from_numpy(be.pack_poses(Rs, tt)).cuda()
        out = torch.empty((nb, 14), dtype=torch.float64, device="cuda")
        be.cascade_batch(W1, W2, False, dom, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision=prec)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            be.cascade_batch(W1, W2, False, dom, 1.0, [0.1, 0.2, 0.3], poses, out=out, precision=prec)
        e1.record(); torch.cuda.synchronize()
        per_pose_us = e0.elapsed_time(e1) * 1e3 / (3 * nb)
        tflops = 240 * w ** 3 / (per_pose_us * 1e-6) / 1e12
        print(f"V={VAR} L={L} {prec} w={w:4d} m'={w**3:8d}  host-query p50={p50:7.1f}us p99={p99:7.1f}us  "
              f"serial-dev={ser_us:7.2f}us/q  batch={per_pose_us:8.3f}us/pose ({1e6/per_pose_us:9.0f} poses/s, {tflops:5.1f} TF@240)", flush=True)
