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
};

void set_error(const std::string& msg);
const char* last_error();

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

template <typename T> struct cx { T re, im; };

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

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace gf
