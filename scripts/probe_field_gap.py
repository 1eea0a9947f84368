import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
exec(open(os.path.join(ROOT, 'scripts/prof_field.py')).read().split('for _ in range(3)')[0])
f = lambda: score_field_device(A(C1), A(C2), R, None, precision=32)
f(); torch.cuda.synchronize()
for _ in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0.record(); f(); t1 = time.perf_counter(); e1.record(); e1.synchronize(); t2 = time.perf_counter()
    print(f"host issue {1e3*(t1-t0):.3f} ms  gpu {e0.elapsed_time(e1):.3f} ms  wall {1e3*(t2-t0):.3f} ms")
import ctypes
from paper_1711_05017_b200 import _lib
g = A(C1).grid
dtype = torch.complex64
N = list(g.dims); w = list(C1.shape)
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    work = torch.empty(max(w[0] * N[1] * N[2], int(np.prod(w))), dtype=dtype, device="cuda")
    work2 = torch.empty(w[0] * w[1] * N[2], dtype=dtype, device="cuda")
    out = torch.empty(g.node_count, dtype=dtype, device="cuda")
    t1 = time.perf_counter()
    dom = np.ascontiguousarray(g.delta_omega(), dtype=np.float64); c = g.center()
    s = np.ascontiguousarray(R @ c - c + np.asarray(g.origin), dtype=np.float64)
    dims = (ctypes.c_int32 * 3)(*N)
    st = torch.cuda.current_stream().cuda_stream
    t2 = time.perf_counter()
    _lib.check(_lib.LIB.gf_score_field(C1.handle, C2.handle, 1, _lib.dptr(dom), dims, _lib.dptr(np.ascontiguousarray(R)), _lib.dptr(s), 1.0, 32, ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(work2.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st)))
    t3 = time.perf_counter()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"alloc {1e3*(t1-t0):.3f}  prep {1e3*(t2-t1):.3f}  gf_score_field {1e3*(t3-t2):.3f}  sync {1e3*(t4-t3):.3f} ms")
    del work, work2, out
print("--- per call host time")
L = _lib.LIB
for _ in range(3):
    work = torch.empty(max(w[0] * N[1] * N[2], int(np.prod(w))), dtype=dtype, device="cuda")
    work2 = torch.empty(w[0] * w[1] * N[2], dtype=dtype, device="cuda")
    out = torch.empty(g.node_count, dtype=dtype, device="cuda")
    torch.cuda.synchronize()
    sh = lambda *v: (ctypes.c_int32 * 3)(*v)
    ts = [time.perf_counter()]
    _lib.check(L.gf_rotate_product(C1.handle, C2.handle, 1, _lib.dptr(dom), _lib.dptr(np.ascontiguousarray(R)), _lib.dptr(s), 32, ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(st))); ts.append(time.perf_counter())
    _lib.check(L.gf_fft_pass(32, ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(work2.data_ptr()), sh(512,512,512), sh(512,512,512), 2, 512, 1, 0, 1, 0.0, 0.0, 1.0, ctypes.c_void_p(st))); ts.append(time.perf_counter())
    _lib.check(L.gf_fft_pass(32, ctypes.c_void_p(work2.data_ptr()), ctypes.c_void_p(work.data_ptr()), sh(512,512,512), sh(512,512,512), 1, 512, 1, 0, 1, 0.0, 0.0, 1.0, ctypes.c_void_p(st))); ts.append(time.perf_counter())
    _lib.check(L.gf_fft_pass(32, ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(out.data_ptr()), sh(512,512,512), sh(512,512,512), 0, 512, 1, 0, 1, 0.0, 0.0, 1.0, ctypes.c_void_p(st))); ts.append(time.perf_counter())
    torch.cuda.synchronize(); ts.append(time.perf_counter())
    print("  ".join(f"{1e3*(b-a):.3f}" for a, b in zip(ts, ts[1:])), "ms (product, z, y, x, sync)")
    del work, work2, out
