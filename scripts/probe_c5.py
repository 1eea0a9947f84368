"""C5 haptic loop (bench.py's setup): per-frame latencies, where the slow frames fall."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_1711_05017_b200 import backend, _lib
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.haptic import HapticSession
_lib.ensure_device(0)
gen = torch.Generator(device="cuda").manual_seed(0)
def mk(w):
    return torch.randn((w,) * 3, dtype=torch.complex128, device="cuda", generator=gen) * 1e-2
n5, w5, dom5 = 256, 128, 4.37
g5 = SampleGrid(3, (n5,) * 3, (-0.5 * dom5,) * 3, dom5 / n5)
f5 = bench._Asset(g5, backend.DeviceWindow(mk(w5)), False), bench._Asset(g5, backend.DeviceWindow(mk(w5)), False)
frames = 1000
th = np.linspace(0.0, 4.0 * np.pi, frames)
R5 = np.stack([bench.axis_rot(2, a) for a in th])
t5 = np.stack([np.array([0.0, 0.0, 0.3 - 0.1 * a / (2 * np.pi)]) for a in th])
sess = HapticSession(f5[0], f5[1], None)
sess.run(R5[:50], t5[:50], rate_hz=1000.0)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    r = sess.run(R5, t5, rate_hz=1000.0)
    print(rep, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()})

# host-only pacing (no GPU work): does the host thread itself stall?
def host_only(n=5000, period=1e-3):
    lat, t_next = [], time.perf_counter()
    for i in range(n):
        t0 = time.perf_counter()
        x = 0
        for _ in range(200):
            x += 1
        lat.append((time.perf_counter() - t0) * 1e6)
        t_next += period
        while time.perf_counter() < t_next:
            pass
    lat.sort()
    return f"host-only p50 {lat[len(lat)//2]:.1f} p99 {lat[int(.99*len(lat))]:.1f} max {lat[-1]:.1f} >1ms {sum(l > 1000 for l in lat)}"
print(host_only())
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
try:
    os.sched_setaffinity(0, {max(os.sched_getaffinity(0))})
    print("pinned to", os.sched_getaffinity(0))
except Exception as e:
    print("affinity failed", e)
try:
    os.sched_setscheduler(0, os.SCHED_FIFO, os.sched_param(50))
    print("SCHED_FIFO ok")
except Exception as e:
    print("fifo failed", e)
print(host_only())
for rep in range(3):
    r = sess.run(R5, t5, rate_hz=1000.0)
    print("pinned", rep, {k: (round(v, 1) if isinstance(v, float) else v) for k, v in r.items()})
