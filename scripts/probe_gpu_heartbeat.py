"""Heartbeat: one warp per SM spins on %globaltimer for a fixed time with no
host interaction and counts gaps longer than a threshold between consecutive
reads (a GPU-wide stall shows on every SM at the same time)."""
import sys, os, ctypes, time
import numpy as np
import torch
from cuda.bindings import nvrtc, driver as cu

src = r'''
extern "C" __global__ void hb(unsigned long long dur_ns, unsigned long long thr_ns, unsigned long long* out,
                              const unsigned long long* host_word) {
  unsigned long long t0, t, prev, maxgap = 0, n = 0, first = 0, sink = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  prev = t0;
  do {
    if (host_word && blockIdx.x == 0) {  // PCIe reads of host-mapped memory, as the server's poller
      unsigned long long v;
      asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(host_word + threadIdx.x) : "memory");
      sink += v;
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned long long g = t - prev;
    if (g > maxgap) maxgap = g;
    if (g > thr_ns) { ++n; if (!first) first = prev - t0; }
    prev = t;
  } while (t - t0 < dur_ns);
  if (sink == 12345) out[0] = 0;
  if (threadIdx.x == 0) { out[3 * blockIdx.x] = maxgap; out[3 * blockIdx.x + 1] = n; out[3 * blockIdx.x + 2] = first; }
}
'''
torch.cuda.init(); torch.zeros(1, device="cuda")
dev = torch.cuda.current_device()
prog = nvrtc.nvrtcCreateProgram(src.encode(), b"hb.cu", 0, [], [])[1]
opts = [b"--gpu-architecture=sm_100a"]
err, = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
size = nvrtc.nvrtcGetCUBINSize(prog)[1]
cubin = bytearray(size); nvrtc.nvrtcGetCUBIN(prog, cubin)
mod = cu.cuModuleLoadData(bytes(cubin))[1]
fn = cu.cuModuleGetFunction(mod, b"hb")[1]
nsm = torch.cuda.get_device_properties(dev).multi_processor_count
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
host = torch.zeros(64, dtype=torch.int64).pin_memory()
for mode in ("idle", "pcie-poll"):
    out = torch.zeros(3 * nsm, dtype=torch.int64, device="cuda")
    dur = ctypes.c_ulonglong(int(secs * 1e9)); thr = ctypes.c_ulonglong(500_000); ptr = ctypes.c_void_p(out.data_ptr())
    hp = ctypes.c_void_p(host.data_ptr() if mode == "pcie-poll" else 0)
    args = (ctypes.c_void_p * 4)(ctypes.addressof(dur), ctypes.addressof(thr), ctypes.addressof(ptr), ctypes.addressof(hp))
    cu.cuLaunchKernel(fn, nsm, 1, 1, 32, 1, 1, 0, 0, ctypes.addressof(args), 0)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(-1, 3)
    print(f"{mode}: {secs:.0f} s, {nsm} SMs: max gap {o[:,0].max()/1e3:.1f} us, gaps > 500 us per SM: min {o[:,1].min()} "
          f"max {o[:,1].max()}, first gap at {o[:,2].min()/1e9:.3f}-{o[:,2].max()/1e9:.3f} s", flush=True)
