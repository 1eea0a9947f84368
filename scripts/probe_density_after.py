import sys, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from paper_1711_05017_b200 import scenes, backend as be, _lib
from paper_1711_05017_b200.descriptor import affinity_field
from conftest import synthetic_window
sc = scenes.get_scene("peg_in_hole"); gd = sc.grid(64)
def dens(tag):
    affinity_field(sc.fixed, gd, sc.kernel); torch.cuda.synchronize()
    t0 = time.perf_counter(); affinity_field(sc.fixed, gd, sc.kernel); print(tag, 1e3 * (time.perf_counter() - t0), "ms", flush=True)
dens("fresh")
rng = np.random.default_rng(0)
W1, W2 = be.DeviceWindow(synthetic_window(rng, 64)), be.DeviceWindow(synthetic_window(rng, 64))
with be.HapticServer(W1, W2, False, (0.1,) * 3, 1.0, [0.1, 0.2, 0.3]):
    be.cascade(W1, W2, False, (0.1,) * 3, 1.0, np.eye(3), np.zeros(3), [0.1, 0.2, 0.3])
dens("after server 1"); dens("after server 2"); dens("after server 3")
import ctypes
pk = ctypes.c_double(); _lib.check(_lib.LIB.gf_measure_fma_peak(32, ctypes.byref(pk))); print("fma TF", pk.value)
import subprocess; print(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active", "--format=csv"], capture_output=True, text=True).stdout)
x = torch.empty(int(6e9) // 8, dtype=torch.float64, device="cuda"); del x; torch.cuda.empty_cache()
dens("after 6GB alloc")
