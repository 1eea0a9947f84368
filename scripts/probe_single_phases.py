import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be, _lib
from conftest import synthetic_window, random_rotation
_lib.ensure_device(0)
rng = np.random.default_rng(0)
for w in [int(x) for x in (sys.argv[1:] or ["32", "64"])]:
    C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
    W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
    dbg = torch.zeros(8 * 2048, dtype=torch.int64, device="cuda")
    n = 20
    Rs = np.stack([random_rotation(rng) for _ in range(n)]); tt = rng.uniform(-1, 1, (n, 3))
    poses = torch.from_numpy(be.pack_poses(Rs, tt)).cuda()
    out = torch.empty((n, 14), dtype=torch.float64, device="cuda")
    be.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses, out=out, serial=True)
    torch.cuda.synchronize()
    _lib.check(_lib.LIB.gf_set_cascade_debug(ctypes.c_void_p(dbg.data_ptr())))
    be.cascade_batch(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3], poses[:1], out=out[:1], serial=True)
    torch.cuda.synchronize()
    _lib.check(_lib.LIB.gf_set_cascade_debug(None))
    d = dbg.cpu().numpy().reshape(-1, 8)
    nb = int(np.count_nonzero(d[:, 0]))
    d = d[:nb].astype(np.float64)
    t0 = d[:, 0].min()
    print(f"w={w} blocks={nb}")
    for k, name in enumerate(["start", "setup_done", "modes_done", "block_reduced", "ticket", "final"]):
        col = d[:, k]
        col = col[col > 0]
        if len(col):
            print(f"  {name:14s} min {1e-3*(col.min()-t0):8.2f} us  med {1e-3*(np.median(col)-t0):8.2f}  max {1e-3*(col.max()-t0):8.2f}")


# persistent server: phases of the last query, relative to the first CTA that saw it
w = 64
C1, C2 = synthetic_window(rng, w), synthetic_window(rng, w)
W1, W2 = be.DeviceWindow(C1), be.DeviceWindow(C2)
dbg = torch.zeros(8 * 2048, dtype=torch.int64, device="cuda")
_lib.check(_lib.LIB.gf_set_cascade_debug(ctypes.c_void_p(dbg.data_ptr())))
with be.HapticServer(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3]):
    for i in range(50):
        be.cascade(W1, W2, False, (0.1,) * 3, 1.0, random_rotation(rng), rng.uniform(-1, 1, 3), [0.1, 0.2, 0.3])
    d = dbg.cpu().numpy().reshape(-1, 8)
_lib.check(_lib.LIB.gf_set_cascade_debug(None))
nb = int(np.count_nonzero(d[:, 7]))
d = d[:nb].astype(np.float64)
t0 = d[:, 7].min()
print(f"server w={w} blocks={nb}")
for k, name in [(7, "seq_seen"), (0, "start"), (1, "setup_done"), (2, "modes_done"), (3, "block_reduced"), (4, "ticket"), (5, "final")]:
    col = d[:, k]
    col = col[col > 0]
    if len(col):
        print(f"  {name:14s} min {1e-3*(col.min()-t0):8.2f} us  med {1e-3*(np.median(col)-t0):8.2f}  max {1e-3*(col.max()-t0):8.2f}")
