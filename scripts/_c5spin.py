import json, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1711_05017_b200 import _lib, backend, haptic
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.haptic import HapticSession
_lib.ensure_device(0)
frames = 5000
w, n = 128, 256
g = SampleGrid(3, (n,) * 3, (-2.185,) * 3, 4.37 / n)
W1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda") * 1e-2)
W2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda") * 1e-2)
class A:
    def __init__(s, win): s.grid, s.w = g, win
    def window(s, m=None): return s.w, False
    def max_modes(s): return w ** 3
th = np.linspace(0.0, 4.0 * np.pi, frames)
R = np.stack([np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]]) for a in th])
t = np.stack([np.array([0.0, 0.0, 0.3 - 0.1 * a / (2 * np.pi)]) for a in th])
sess = HapticSession(A(W1), A(W2), None)
sess.run(R[:200], t[:200])
for spin in (150e-6, 400e-6, 700e-6, 150e-6):
    haptic._SPIN_S = spin
    for rt in (True, False):
        out = sess.run(R, t, realtime=rt)
        print(f"spin {spin*1e6:.0f} us realtime {rt}: p50 {out['p50_us']:.1f} p99 {out['p99_us']:.1f} max {out['max_us']:.0f} gpu {out['gpu_us_p50']:.1f} misses {out['deadline_misses']}", flush=True)
