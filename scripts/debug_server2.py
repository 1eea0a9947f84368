import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1711_05017_b200 import backend as be
from conftest import synthetic_window, random_rotation
rng = np.random.default_rng(21)
for w, wrap in ((32, False), (16, True)):
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, c = (0.11, 0.11, 0.11), np.array([0.1, 0.2, -0.3])
    poses = [(random_rotation(rng), rng.uniform(-1, 1, 3)) for _ in range(5)]
    want = [be.cascade(W1, W2, wrap, dom, 0.4, R, t, c) for R, t in poses]
    print("want ok", w, flush=True)
    t0 = time.time()
    with be.HapticServer(W1, W2, wrap, dom, 0.4, c, idle_timeout_s=3.0) as srv:
        print("server", srv.id, "started", time.time() - t0, "matches", srv.matches(0.4, np.array(dom), c), flush=True)
        for i, (R, t) in enumerate(poses):
            g = be.cascade(W1, W2, wrap, dom, 0.4, R, t, c)
            print(i, time.time() - t0, np.max(np.abs(g - want[i])), flush=True)
    print("stopped", time.time() - t0, flush=True)
