"""Decompose the single-query end-to-end time (headline C2, w=64, fp32)."""
import os, sys, time, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_1711_05017_b200 import backend as be, _lib
from conftest import synthetic_window, random_rotation
_lib.ensure_device(0)
if os.environ.get('GF_PREC'):
    be.set_precision(os.environ['GF_PREC'])
if os.environ.get('GF_TILE'):
    _lib.check(_lib.LIB.gf_set_cascade_tile(int(os.environ['GF_TILE'])))
rng = np.random.default_rng(0)
w = int(sys.argv[1]) if len(sys.argv) > 1 else 64
W1, W2 = be.DeviceWindow(synthetic_window(rng, w)), be.DeviceWindow(synthetic_window(rng, w))
n = 3000
Rs = np.stack([random_rotation(rng) for _ in range(n)]); ts = rng.uniform(-1, 1, (n, 3))
dom = (0.1,) * 3; cen = np.array([0.1, 0.2, 0.3])
def pct(x):
    x = np.sort(np.asarray(x)); return f"p50 {np.median(x):6.2f}  p90 {x[int(.9*len(x))]:6.2f}  p99 {x[int(.99*len(x))]:6.2f} us"
for _ in range(200): be.cascade(W1, W2, False, dom, 1.0, Rs[0], ts[0], cen)
lat = []
for i in range(n):
    t0 = time.perf_counter(); be.cascade(W1, W2, False, dom, 1.0, Rs[i], ts[i], cen); lat.append((time.perf_counter() - t0) * 1e6)
print("A backend.cascade         ", pct(lat))
q = be._qb
q.arg[12:15] = cen; q.arg[15:18] = dom
f = _lib.LIB.gf_cascade_fast
lat = []
for i in range(n):
    q.arg[:9] = Rs[i].ravel(); q.arg[9:12] = ts[i]
    t0 = time.perf_counter(); f(W1.handle, W2.handle, 0, q.pd, 1.0, q.pR, q.pt, q.pc, 64 if be.precision() == 'fp64' else 32, q.pout); lat.append((time.perf_counter() - t0) * 1e6)
print("B raw gf_cascade (ctypes) ", pct(lat))
lat = []
for i in range(n):
    t0 = time.perf_counter(); lat.append((time.perf_counter() - t0) * 1e6)
print("  perf_counter pair        ", pct(lat))
for blocks in (1, 296):
    h, d = ctypes.c_double(), ctypes.c_double()
    _lib.check(_lib.LIB.gf_measure_launch(2000, blocks, ctypes.byref(h), ctypes.byref(d)))
    print(f"C empty kernel blocks={blocks:4d}: host {h.value:6.2f} us/launch  device {d.value:6.2f} us/launch")
poses = torch.from_numpy(be.pack_poses(Rs[:1000], ts[:1000])).cuda()
out = torch.empty((1000, 14), dtype=torch.float64, device="cuda")
be.cascade_batch(W1, W2, False, dom, 1.0, cen, poses, out=out, serial=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
be.cascade_batch(W1, W2, False, dom, 1.0, cen, poses, out=out, serial=True)
e1.record(); torch.cuda.synchronize()
print(f"D device serial loop: {e0.elapsed_time(e1) * 1e3 / 1000:6.2f} us/query")
with be.HapticServer(W1, W2, False, dom, 1.0, cen) as srv:
    for _ in range(200): be.cascade(W1, W2, False, dom, 1.0, Rs[0], ts[0], cen)
    lat = []
    for i in range(n):
        t0 = time.perf_counter(); be.cascade(W1, W2, False, dom, 1.0, Rs[i], ts[i], cen); lat.append((time.perf_counter() - t0) * 1e6)
    print("E server backend.cascade  ", pct(lat))
    fq = _lib.LIB.gf_server_query_fast
    lat = []
    for i in range(n):
        q.arg[:9] = Rs[i].ravel(); q.arg[9:12] = ts[i]
        t0 = time.perf_counter(); fq(srv.id, q.pR, q.pt, q.pout); lat.append((time.perf_counter() - t0) * 1e6)
    print("F server raw query        ", pct(lat))
# G: the C5-style call chain -- evaluate() in a haptic_session on stub assets
from paper_1711_05017_b200.descriptor import SampleGrid
from paper_1711_05017_b200.energy import Configuration, evaluate, haptic_session
N = 2 * w
g = SampleGrid(3, (N,) * 3, (-2.0,) * 3, 4.0 / N)


class _A:
    def __init__(s, win): s.grid, s.win, s.vector = g, win, None
    def window(s, m=None): return s.win, False
    def max_modes(s): return w ** 3


a1, a2 = _A(W1), _A(W2)
cfgs = [Configuration(Rs[i], ts[i]) for i in range(n)]
with haptic_session(a1, a2):
    for i in range(200): evaluate(a1, a2, cfgs[i])
    lat = []
    for i in range(n):
        t0 = time.perf_counter(); evaluate(a1, a2, cfgs[i]); lat.append((time.perf_counter() - t0) * 1e6)
    print("G session evaluate()      ", pct(lat))
    lat = []
    for i in range(n):
        t0 = time.perf_counter(); evaluate(a1, a2, Configuration(Rs[i], ts[i])); lat.append((time.perf_counter() - t0) * 1e6)
    print("H + Configuration()       ", pct(lat))
    # I: the same call paced at a fixed period (busy wait between frames)
    for period_us in (100.0, 1000.0):
        lat = []
        t_next = time.perf_counter()
        for i in range(1000):
            t0 = time.perf_counter(); evaluate(a1, a2, cfgs[i]); lat.append((time.perf_counter() - t0) * 1e6)
            t_next += period_us * 1e-6
            while time.perf_counter() < t_next:
                pass
        print(f"I paced every {period_us:6.0f} us   ", pct(lat))
    # K: rotations about z (the C5 screw): mode z maps onto C2 z exactly -> index ties on every mode
    def zrot(a):
        c, s_ = np.cos(a), np.sin(a)
        return np.array([[c, -s_, 0.0], [s_, c, 0.0], [0.0, 0.0, 1.0]])
    zc = [Configuration(zrot(a), np.array([0.0, 0.0, 0.3 - 0.1 * a / (2 * np.pi)])) for a in np.linspace(0, 4 * np.pi, n)]
    for i in range(200): evaluate(a1, a2, zc[i])
    lat = []
    for i in range(n):
        t0 = time.perf_counter(); evaluate(a1, a2, zc[i]); lat.append((time.perf_counter() - t0) * 1e6)
    print("K evaluate, z-axis screw  ", pct(lat))
    ic = [Configuration(np.eye(3), ts[i]) for i in range(n)]
    lat = []
    for i in range(n):
        t0 = time.perf_counter(); evaluate(a1, a2, ic[i]); lat.append((time.perf_counter() - t0) * 1e6)
    print("L evaluate, identity R    ", pct(lat))
