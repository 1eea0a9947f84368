"""Probe: resident-server latency vs SM budget (headline C2, w=64, fp32):
host round trip and GPU detect->result per query, p50 over 3000 queries."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from paper_1711_05017_b200 import backend as be, _lib
from conftest import synthetic_window, random_rotation
_lib.ensure_device(0)
rng = np.random.default_rng(0)
w = int(sys.argv[1]) if len(sys.argv) > 1 else 64
W1, W2 = be.DeviceWindow(synthetic_window(rng, w)), be.DeviceWindow(synthetic_window(rng, w))
n = 3000
Rs = np.stack([random_rotation(rng) for _ in range(n)]); ts = rng.uniform(-1, 1, (n, 3))
dom = (0.1,) * 3; cen = (0.1, 0.2, 0.3)
for sms in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,128,96,64,48,32,16".split(","))]:
    with be.HapticServer(W1, W2, False, dom, 1.0, cen, max_sms=sms) as srv:
        for i in range(300): be.cascade(W1, W2, False, dom, 1.0, Rs[i], ts[i], cen)
        host, gpu, p2d, r2h = [], [], [], []
        for i in range(n):
            t0 = time.perf_counter(); be.cascade(W1, W2, False, dom, 1.0, Rs[i], ts[i], cen)
            host.append((time.perf_counter() - t0) * 1e6)
            lt = srv.last_timing(); gpu.append(lt["gpu_us"]); p2d.append(lt["post_to_detect_us"]); r2h.append(lt["result_to_host_us"])
        med = lambda x: float(np.median(x))
        print(f"max_sms={sms:4d}  host p50 {med(host):6.2f}  gpu p50 {med(gpu):6.2f}  post->detect {med(p2d):5.2f}  "
              f"result->host {med(r2h):5.2f} us", flush=True)
