"""fp64 resident server vs launch path: bit equality at w=64/96."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_1711_05017_b200 import backend as be
from conftest import synthetic_window, random_rotation
rng = np.random.default_rng(5096)
for w in (64, 96):
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dom, dcell, c = (0.07,) * 3, 0.21, rng.normal(size=3)
    poses = [(random_rotation(rng), rng.uniform(-2, 2, 3)) for _ in range(2)]
    got = [be.cascade(W1, W2, False, dom, dcell, R, t, c, precision="fp64") for R, t in poses]
    with be.HapticServer(W1, W2, False, dom, dcell, c, precision="fp64"):
        srv = [be.cascade(W1, W2, False, dom, dcell, R, t, c, precision="fp64") for R, t in poses]
    print(os.environ.get("GF_SINGLE_CLUSTER"), w, [bool(np.array_equal(a, b)) for a, b in zip(srv, got)])
