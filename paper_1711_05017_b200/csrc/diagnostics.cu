// diagnostics.cu -- roofline denominators measured on the device itself.
//
// MEASURED_PEAKS.json carries HBM copy bandwidth and cuBLAS bf16 only; the
// query/sweep kernels are bound by the FP32 (or FP64) FMA pipe, so bench.py
// measures that pipe live with this FMA-chain kernel (SURVEY.md section 6
// asks for exactly this measurement).
#include "../../include/geofield_b200.h"
#include "common.cuh"

#include <chrono>

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
