// common.cuh -- shared helpers for the geofield B200 engine (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace gf {

// ---------------------------------------------------------------------------
// error plumbing: every C-ABI entry returns 0 / cudaError_t (>0) / gf error (<0)
// and records a message retrievable with gf_last_error().

enum GfStatus : int {
  GF_OK = 0,
  GF_EINVAL = -1,   // bad argument (shape, handle, dtype)
  GF_ENOMEM = -2,   // host allocation failure
  GF_EINTERNAL = -3,
  GF_ESTOPPED = -4, // haptic server no longer running (stopped / idle timeout)
};

void set_error(const std::string& msg);
const char* last_error();

// cudaFree synchronises the whole device; while a persistent haptic server
// grid is resident that would wait for its idle timeout.  All engine frees go
// through device_free, which defers them until no server is running.
void device_free(void* p);

// Per-device launch plumbing (capi.cu), thread-safe: the attribute and
// occupancy caches are keyed by (kernel, device), so a second device in the
// same process gets its own cudaFuncSetAttribute and SM count.
//   ensure_smem   raise `func`'s dynamic shared-memory limit to >= bytes
//                 (no-op below the 48 KB default) on the current device;
//   sm_count      multiprocessor count of the current device;
//   resident_ctas CTAs of `func` resident per SM at (threads, smem), >= 1.
cudaError_t ensure_smem(const void* func, size_t bytes);
int sm_count();
int resident_ctas(const void* func, int threads, size_t smem);

#define GF_CUDA(expr)                                                            \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::gf::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));       \
      return (int)_e;                                                            \
    }                                                                            \
  } while (0)

#define GF_CHECK(cond, code, msg)                                                \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::gf::set_error(msg);                                                      \
      return (int)(code);                                                        \
    }                                                                            \
  } while (0)

// ---------------------------------------------------------------------------
// complex arithmetic on float2/double2-shaped structs

// 8/16-byte aligned so that loads and stores of one element are single vector
// accesses (a 4-byte-aligned pair splits into two LDG/STG.32).
template <typename T> struct alignas(2 * sizeof(T)) cx { T re, im; };

template <typename T> __host__ __device__ __forceinline__ cx<T> mk(T r, T i) { return cx<T>{r, i}; }
template <typename T> __host__ __device__ __forceinline__ cx<T> operator+(cx<T> a, cx<T> b) {
  return cx<T>{a.re + b.re, a.im + b.im};
}
template <typename T> __host__ __device__ __forceinline__ cx<T> operator-(cx<T> a, cx<T> b) {
  return cx<T>{a.re - b.re, a.im - b.im};
}
template <typename T> __host__ __device__ __forceinline__ cx<T> operator*(cx<T> a, cx<T> b) {
  return cx<T>{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
template <typename T> __host__ __device__ __forceinline__ cx<T> operator*(T s, cx<T> a) {
  return cx<T>{s * a.re, s * a.im};
}
template <typename T> __host__ __device__ __forceinline__ void operator+=(cx<T>& a, cx<T> b) {
  a.re += b.re;
  a.im += b.im;
}
// a += s * b (two FMAs)
template <typename T> __device__ __forceinline__ void axpy(cx<T>& a, T s, cx<T> b) {
  a.re = fma(s, b.re, a.re);
  a.im = fma(s, b.im, a.im);
}
// lerp a + f (b - a)
template <typename T> __device__ __forceinline__ cx<T> lerp(cx<T> a, cx<T> b, T f) {
  return cx<T>{fma(f, b.re - a.re, a.re), fma(f, b.im - a.im, a.im)};
}

// vector type carrying two consecutive complex values (one packed corner pair)
template <typename T> struct pair4;
template <> struct pair4<float> { using type = float4; };
template <> struct pair4<double> { using type = double4; };

// read-only 16/32-byte loads of a packed corner pair
__device__ __forceinline__ float4 ldg_pair(const float4* p) { return __ldg(p); }
__device__ __forceinline__ double4 ldg_pair(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 lo = __ldg(q), hi = __ldg(q + 1);
  return make_double4(lo.x, lo.y, hi.x, hi.y);
}

// ---------------------------------------------------------------------------
// 32.32 fixed-point continuous window index (fp32 engine).
//
// u = h + sum_b mu[a][b] kappa_b is formed exactly in int64 from fixed-point
// coefficients (|error| < 1e-7 for windows up to 1024), so floor(u) comes
// from a shift and frac(u) from the low word, with no float rounding of a
// large |u| -- the near-integer band that must be re-decided in float64
// reference order shrinks from ~1e-4 to 1e-6 and the conversion pipe is not
// used.  Non-negative and negative u both floor correctly (arithmetic shift).
__host__ __device__ __forceinline__ long long to_fix32(double x) {
  return (long long)llrint(x * 4294967296.0);
}
constexpr unsigned kFixTieEps = 4295u;  // 1e-6 in units of 2^-32
__device__ __forceinline__ int fix_floor(long long u) { return (int)(u >> 32); }
__device__ __forceinline__ unsigned fix_lo(long long u) { return (unsigned)((unsigned long long)u & 0xffffffffull); }
__device__ __forceinline__ float fix_frac(unsigned lo) { return __uint_as_float(0x3f800000u | (lo >> 9)) - 1.0f; }
// lo < eps or lo > 2^32 - 1 - eps, as one wrapped compare
__device__ __forceinline__ bool fix_tie(unsigned lo) { return lo + kFixTieEps < 2u * kFixTieEps; }

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace gf
