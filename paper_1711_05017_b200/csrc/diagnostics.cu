// diagnostics.cu -- roofline denominators measured on the device itself.
//
// MEASURED_PEAKS.json carries HBM copy bandwidth and cuBLAS bf16 only; the
// query/sweep kernels are bound by the FP32 (or FP64) FMA pipe, so bench.py
// measures that pipe live with this FMA-chain kernel (SURVEY.md section 6
// asks for exactly this measurement).
#include "../../include/geofield_b200.h"
#include "common.cuh"

#include <chrono>
#include <cstring>

namespace gf {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) fma_chain_kernel(T* sink, int iters, T a, T b) {
  // 16 independent accumulator chains per thread keep the FMA pipe full
  T x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == (T)1234.5678) sink[0] = s;  // keep the chains live
}

}  // namespace
}  // namespace gf

extern "C" int gf_measure_fma_peak(int precision, double* tflops) {
  using namespace gf;
  GF_CHECK(tflops != nullptr, GF_EINVAL, "null argument");
  GF_CHECK(precision == 32 || precision == 64, GF_EINVAL, "precision must be 32 or 64");
  int dev = 0, sms = 0;
  GF_CUDA(cudaGetDevice(&dev));
  GF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* sink = nullptr;
  GF_CUDA(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1;
  GF_CUDA(cudaEventCreate(&e0));
  GF_CUDA(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  const int iters = precision == 32 ? 16384 : 4096;
  float best_ms = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    GF_CUDA(cudaEventRecord(e0));
    if (precision == 32)
      fma_chain_kernel<float><<<blocks, threads>>>((float*)sink, iters, 0.999999f, 1e-7f);
    else
      fma_chain_kernel<double><<<blocks, threads>>>((double*)sink, iters, 0.999999, 1e-7);
    GF_CUDA(cudaEventRecord(e1));
    GF_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    GF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (rep > 0 && ms < best_ms) best_ms = ms;
  }
  double flops = 2.0 * 16.0 * iters * (double)blocks * threads;
  *tflops = flops / (best_ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return 0;
}

namespace gf {
namespace {
__global__ void empty_kernel(int* p) {
  if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] = 1;
}
}  // namespace
}  // namespace gf

// Launch-overhead probe: n back-to-back empty launches of `blocks` CTAs on a
// fresh stream; returns host microseconds per launch and device microseconds
// per launch (events around the whole sequence).
extern "C" int gf_measure_launch(int n, int blocks, double* host_us, double* dev_us) {
  using namespace gf;
  GF_CHECK(n > 0 && host_us && dev_us, GF_EINVAL, "bad argument");
  cudaStream_t st;
  GF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  GF_CUDA(cudaEventCreate(&e0));
  GF_CUDA(cudaEventCreate(&e1));
  empty_kernel<<<blocks, 256, 0, st>>>(nullptr);
  GF_CUDA(cudaStreamSynchronize(st));
  auto t0 = std::chrono::steady_clock::now();
  GF_CUDA(cudaEventRecord(e0, st));
  for (int i = 0; i < n; ++i) empty_kernel<<<blocks, 256, 0, st>>>(nullptr);
  GF_CUDA(cudaEventRecord(e1, st));
  auto t1 = std::chrono::steady_clock::now();
  GF_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  GF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *host_us = std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
  *dev_us = 1e3 * ms / n;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  return 0;
}

// ---------------------------------------------------------------------------
// Host <-> device round-trip probe for the single-query path design.
namespace gf {
namespace {
__global__ void signal_kernel(volatile unsigned* done, unsigned v) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    __threadfence_system();
    *done = v;
  }
}
// dependent reads of a host-mapped word, and mapped write + system fence
__global__ void pcie_latency_kernel(volatile unsigned* hostw, int n, unsigned long long* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long t0, t1, t2;
  unsigned acc = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < n; ++i) acc += hostw[acc & 1];
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  for (int i = 0; i < n; ++i) {
    hostw[2] = acc + i;
    __threadfence_system();
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
  out[0] = (t1 - t0) / n;
  out[1] = (t2 - t1) / n;
  out[2] = acc;
}
}  // namespace
}  // namespace gf

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>

// out[0]: p50 us, launch of a 1-CTA kernel that signals a mapped word, host polls
// out[1]: p50 us, the same kernel pre-enqueued behind cuStreamWaitValue32 on a
//         mapped flag; the host writes the flag and polls (launch off the path)
// out[2]: GPU read latency of host-mapped memory, ns (dependent reads)
// out[3]: GPU mapped write + __threadfence_system, ns
extern "C" int gf_measure_roundtrip(int n, double* out) {
  using namespace gf;
  GF_CHECK(out && n > 0, GF_EINVAL, "bad argument");
  cudaStream_t st;
  GF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  unsigned* h = nullptr;
  GF_CUDA(cudaHostAlloc((void**)&h, 4096, cudaHostAllocMapped));
  std::memset(h, 0, 4096);
  unsigned* d = nullptr;
  GF_CUDA(cudaHostGetDevicePointer((void**)&d, h, 0));
  volatile unsigned* done = h;       // word 0: completion
  volatile unsigned* flag = h + 32;  // word 32: go flag (own line)
  std::vector<double> t(n);
  for (int i = 0; i < n + 50; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    signal_kernel<<<1, 32, 0, st>>>(d, (unsigned)(i + 1));
    while (*done != (unsigned)(i + 1)) {
    }
    auto t1 = std::chrono::steady_clock::now();
    if (i >= 50) t[i - 50] = std::chrono::duration<double, std::micro>(t1 - t0).count();
  }
  std::sort(t.begin(), t.end());
  out[0] = t[n / 2];
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  out[1] = -1.0;
  if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fnp, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess && fnp) {
    auto wait = (PFN_cuStreamWaitValue32_v11070)fnp;
    GF_CUDA(cudaStreamSynchronize(st));
    *done = 0;
    unsigned base = 1000;
    auto arm = [&](unsigned k) -> int {
      if (wait((CUstream)st, (CUdeviceptr)(d + 32), k, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) return 1;
      signal_kernel<<<1, 32, 0, st>>>(d, k);
      return 0;
    };
    GF_CHECK(arm(base + 1) == 0, GF_EINTERNAL, "cuStreamWaitValue32 failed");
    for (int i = 0; i < n + 50; ++i) {
      const unsigned k = base + 1 + i;
      // let the pre-armed pair reach the wait before timing
      auto tw = std::chrono::steady_clock::now();
      while (std::chrono::steady_clock::now() - tw < std::chrono::microseconds(30)) {
      }
      auto t0 = std::chrono::steady_clock::now();
      *flag = k;
      while (*done != k) {
      }
      auto t1 = std::chrono::steady_clock::now();
      if (i >= 50) t[i - 50] = std::chrono::duration<double, std::micro>(t1 - t0).count();
      GF_CHECK(arm(k + 1) == 0, GF_EINTERNAL, "cuStreamWaitValue32 failed");
    }
    *flag = base + n + 100;  // release the last armed pair
    GF_CUDA(cudaStreamSynchronize(st));
    std::sort(t.begin(), t.end());
    out[1] = t[n / 2];
  }
  unsigned long long* dl = nullptr;
  GF_CUDA(cudaMalloc(&dl, 3 * sizeof(unsigned long long)));
  pcie_latency_kernel<<<1, 32, 0, st>>>(d + 64, 200, dl);
  unsigned long long hl[3];
  GF_CUDA(cudaMemcpyAsync(hl, dl, sizeof hl, cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  out[2] = (double)hl[0];
  out[3] = (double)hl[1];
  cudaFree(dl);
  cudaFreeHost(h);
  cudaStreamDestroy(st);
  return 0;
}

// ---------------------------------------------------------------------------
// GPU-wide stall detector: one warp per SM spins on %globaltimer for a fixed
// time with no host interaction and records, per SM, the longest gap between
// consecutive reads and the number of gaps over a threshold.  A stall of the
// whole GPU shows on every SM with the same count (the C5 frame misses).
namespace gf {
namespace {
__global__ void heartbeat_kernel(unsigned long long dur_ns, unsigned long long thr_ns, unsigned long long* out) {
  unsigned long long t0, t, prev, maxgap = 0, n = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  prev = t0;
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long g = t - prev;
    maxgap = g > maxgap ? g : maxgap;
    n += g > thr_ns;
    prev = t;
  } while (t - t0 < dur_ns);
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = maxgap;
    out[2 * blockIdx.x + 1] = n;
  }
}
}  // namespace
}  // namespace gf

// out[0]: longest gap (us) on any SM; out[1]/out[2]: fewest / most gaps over
// threshold_us seen by one SM; out[3]: SMs watched
extern "C" int gf_measure_stalls(double seconds, double threshold_us, double* out) {
  using namespace gf;
  GF_CHECK(out && seconds > 0 && seconds <= 60 && threshold_us > 0, GF_EINVAL, "bad argument");
  const int sms = sm_count();
  unsigned long long* d = nullptr;
  GF_CUDA(cudaMalloc(&d, sizeof(unsigned long long) * 2 * sms));
  cudaStream_t st;
  GF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  heartbeat_kernel<<<sms, 32, 0, st>>>((unsigned long long)(seconds * 1e9), (unsigned long long)(threshold_us * 1e3),
                                       d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  std::vector<unsigned long long> h(2 * sms);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), d, sizeof(unsigned long long) * 2 * sms, cudaMemcpyDeviceToHost);
  cudaStreamDestroy(st);
  cudaFree(d);
  GF_CUDA(e);
  unsigned long long mx = 0, nmin = ~0ull, nmax = 0;
  for (int i = 0; i < sms; ++i) {
    mx = std::max(mx, h[2 * i]);
    nmin = std::min(nmin, h[2 * i + 1]);
    nmax = std::max(nmax, h[2 * i + 1]);
  }
  out[0] = 1e-3 * (double)mx;
  out[1] = (double)nmin;
  out[2] = (double)nmax;
  out[3] = (double)sms;
  return 0;
}
