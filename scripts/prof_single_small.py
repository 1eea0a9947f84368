"""ncu workload: single-query kernels at a given w (default 8)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1711_05017_b200 import backend as be, _lib
from conftest import synthetic_window, random_rotation
_lib.ensure_device(0)
rng = np.random.default_rng(0)
w = int(sys.argv[1]) if len(sys.argv) > 1 else 8
W1, W2 = be.DeviceWindow(synthetic_window(rng, w)), be.DeviceWindow(synthetic_window(rng, w))
for i in range(30):
    be.cascade(W1, W2, False, (0.1,) * 3, 1.0, random_rotation(rng), rng.uniform(-1, 1, 3), [0.1, 0.2, 0.3])
print("ok")
