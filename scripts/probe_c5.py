"""C5 servo loop diagnostics: 10^4 frames of a w=128 screw trajectory at
1 kHz from a resident grid; prints misses with host vs GPU time."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_05017_b200 import _lib, backend  # noqa: E402
from paper_1711_05017_b200.descriptor import SampleGrid  # noqa: E402
from paper_1711_05017_b200.haptic import HapticSession  # noqa: E402

_lib.ensure_device(0)
frames = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
w, n = 128, 256
g = SampleGrid(3, (n,) * 3, (-2.185,) * 3, 4.37 / n)
W1 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda") * 1e-2)
W2 = backend.DeviceWindow(torch.randn((w,) * 3, dtype=torch.complex128, device="cuda") * 1e-2)


class A:
    def __init__(s, win):
        s.grid, s.w = g, win

    def window(s, m=None):
        return s.w, False

    def max_modes(s):
        return w ** 3


th = np.linspace(0.0, 4.0 * np.pi, frames)
R = np.stack([np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1.0]]) for a in th])
t = np.stack([np.array([0.0, 0.0, 0.3 - 0.1 * a / (2 * np.pi)]) for a in th])
sess = HapticSession(A(W1), A(W2), None)
sess.run(R[:200], t[:200])
for rep in range(2):
    out = sess.run(R, t)
    print(json.dumps({k: out[k] for k in ("frames", "p50_us", "p99_us", "max_us", "deadline_misses", "missed",
                                          "realtime", "rt_runtime_us")}), flush=True)
# typical frame for reference (clock offset between host realtime and globaltimer)
from paper_1711_05017_b200.energy import haptic_session  # noqa: E402

with haptic_session(A(W1), A(W2), None) as srv:
    from paper_1711_05017_b200.energy import Configuration, evaluate  # noqa: E402

    rows = []
    for i in range(200):
        evaluate(A(W1), A(W2), Configuration(R[i], t[i]))
        rows.append(srv.last_timing())
    print("typical", json.dumps({k: float(np.median([r[k] for r in rows])) for k in rows[0]}))
# pacing variant: spin through the slack (no sleep; not SCHED_FIFO, which would hit the RT throttle)
import paper_1711_05017_b200.haptic as hp  # noqa: E402

hp._SPIN_S = 1.0
out = sess.run(R, t, realtime=False)
print("spin", json.dumps({k: out[k] for k in ("frames", "p99_us", "max_us", "deadline_misses", "missed")}), flush=True)
