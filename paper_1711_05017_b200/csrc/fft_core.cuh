// fft_core.cuh -- register radix-8 Stockham line FFT used by fft.cu and the
// fused landscape kernel (field.cu).  See fft.cu for the pass semantics.
#pragma once
#include "common.cuh"

namespace gf {

__device__ __forceinline__ cx<float> ldtw(const cx<float>* p) {
  float2 v = __ldg(reinterpret_cast<const float2*>(p));
  return mk<float>(v.x, v.y);
}
__device__ __forceinline__ cx<double> ldtw(const cx<double>* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return mk<double>(v.x, v.y);
}
// multiply by exp(sign * i * pi / 2) = sign * i
template <typename T> __device__ __forceinline__ cx<T> rot90(cx<T> a, int sign) {
  return sign > 0 ? mk<T>(-a.im, a.re) : mk<T>(a.im, -a.re);
}

template <typename T> __device__ __forceinline__ void dft2(cx<T>& a, cx<T>& b) {
  cx<T> t = a - b;
  a = a + b;
  b = t;
}

template <typename T> __device__ __forceinline__ void dft4(cx<T>* v, int sign) {
  // v0..v3 -> X_k = sum v_n exp(sign 2 pi i n k / 4)
  cx<T> a0 = v[0] + v[2], a1 = v[0] - v[2];
  cx<T> b0 = v[1] + v[3], b1 = rot90(v[1] - v[3], sign);
  v[0] = a0 + b0;
  v[2] = a0 - b0;
  v[1] = a1 + b1;
  v[3] = a1 - b1;
}

template <typename T> __device__ __forceinline__ void dft8(cx<T>* v, int sign) {
  const T r = (T)0.70710678118654752440;
  cx<T> e[4] = {v[0], v[2], v[4], v[6]};
  cx<T> o[4] = {v[1], v[3], v[5], v[7]};
  dft4(e, sign);
  dft4(o, sign);
  // twiddles exp(sign 2 pi i k / 8), k = 0..3
  const cx<T> w1 = mk<T>(r, (T)sign * r);
  const cx<T> o1 = o[1] * w1;
  const cx<T> o2 = rot90(o[2], sign);
  const cx<T> o3 = rot90(o[3] * w1, sign);
  v[0] = e[0] + o[0];
  v[4] = e[0] - o[0];
  v[1] = e[1] + o1;
  v[5] = e[1] - o1;
  v[2] = e[2] + o2;
  v[6] = e[2] - o2;
  v[3] = e[3] + o3;
  v[7] = e[3] - o3;
}

template <typename T> __device__ __forceinline__ cx<T> phase_factor(int kind, double ph, int m) {
  if (kind == 1) return (m & 1) ? mk<T>(-1, 0) : mk<T>(1, 0);
  double cyc = ph * (double)m;
  cyc -= rint(cyc);
  double s, c;
  sincospi(2.0 * cyc, &s, &c);
  return mk<T>((T)c, (T)s);
}


// v[r] *= t^r, r = 1..R-1.  One table load per thread and stage (lanes read
// consecutive entries) instead of R-1 strided ones, which made the twiddle
// reads -- not the data -- the L1 bottleneck of contiguous-axis passes; the
// powers by repeated squaring cost < 3 ulp at R = 8.
template <typename T, int R> __device__ __forceinline__ void twiddle_powers(cx<T>* v, cx<T> t) {
  if constexpr (R >= 2) v[1] = v[1] * t;
  if constexpr (R >= 4) {
    const cx<T> t2 = t * t;
    const cx<T> t3 = t2 * t;
    v[2] = v[2] * t2;
    v[3] = v[3] * t3;
    if constexpr (R >= 8) {
      const cx<T> t4 = t2 * t2;
      v[4] = v[4] * t4;
      v[5] = v[5] * (t4 * t);
      v[6] = v[6] * (t3 * t3);
      v[7] = v[7] * (t4 * t3);
    }
  }
}

// Shared-memory line layout: one pad element every 128 bytes, so the
// stride-8 stores of the first radix-8 stage (positions 8 j + r) spread over
// the banks instead of piling onto two of them.
template <typename T> __device__ __forceinline__ int sidx(int i) {
  return i + i / (int)(128 / sizeof(cx<T>));
}
template <typename T, int N> struct LineLD {
  static constexpr int value = N + N / (int)(128 / sizeof(cx<T>)) + 1;
};

template <int N> struct FftShape {
  static constexpr int TPL = N >= 8 ? N / 8 : 1;  // threads per line
  static constexpr int PT = N >= 8 ? 8 : N;       // points per thread
  static constexpr int n_r8 = N >= 8 ? (N <= 8 ? 1 : N <= 32 ? 1 : N <= 256 ? 2 : N <= 2048 ? 3 : 4) : 0;
  static constexpr int pow8 = n_r8 == 0 ? 1 : n_r8 == 1 ? 8 : n_r8 == 2 ? 64 : n_r8 == 3 ? 512 : 4096;
  static constexpr int rest = N >= 8 ? N / pow8 : N;  // final radix (1: none, 2 or 4)
};

// Transform one line.  On entry v[r] holds FFT input position j + r * TPL of
// this thread; on exit the natural-order result is in line[0..N) (all
// threads of the line synchronised).  `line` is this line's shared buffer.
// Element i of a line: padded private line (RS = 0), or row i of a [row][RS]
// tile whose lines are its columns (RS > 0: lanes of a warp walk the columns,
// so every access pattern below is a full, conflict-free 128-byte row).
template <typename T, int RS> __device__ __forceinline__ int lidx(int i) { return RS ? i * RS : sidx<T>(i); }

template <typename T, int N, int RS = 0>
__device__ __forceinline__ void fft_line(cx<T>* v, cx<T>* line, int j, const cx<T>* __restrict__ tw, int sign) {
  using S = FftShape<N>;
  constexpr int TPL = S::TPL, PT = S::PT;
  int Ns = 1;
#pragma unroll
  for (int s = 0; s < S::n_r8; ++s) {
    if (s > 0) {
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = line[lidx<T, RS>(j + r * TPL)];
    }
    const int k = j & (Ns - 1);
    if (Ns > 1) twiddle_powers<T, 8>(v, ldtw(&tw[k * (N / (Ns * 8))]));
    dft8(v, sign);
    const int idx = (j - k) * 8 + k;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) line[lidx<T, RS>(idx + r * Ns)] = v[r];
    Ns *= 8;
  }
  if constexpr (S::rest == 4 || S::rest == 2) {
    constexpr int R = S::rest;
    constexpr int per = PT / R;
    if constexpr (S::n_r8 > 0) {
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = line[lidx<T, RS>(j + r * TPL)];
    }
    cx<T> w[PT];
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const int jj = j + q * TPL;
      cx<T> u[R];
#pragma unroll
      for (int r = 0; r < R; ++r) u[r] = v[q + r * per];
      const int k = jj & (Ns - 1);
      if (Ns > 1) twiddle_powers<T, R>(u, ldtw(&tw[k * (N / (Ns * R))]));
      if constexpr (R == 4) dft4(u, sign);
      else dft2(u[0], u[1]);
#pragma unroll
      for (int r = 0; r < R; ++r) w[q * R + r] = u[r];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < per; ++q) {
      const int jj = j + q * TPL;
      const int k = jj & (Ns - 1);
#pragma unroll
      for (int r = 0; r < R; ++r) line[lidx<T, RS>((jj - k) * R + k + r * Ns)] = w[q * R + r];
    }
  }
  __syncthreads();
}

// Twiddle table W_N^m = exp(sign 2 pi i m / N), m < N (device, cached per
// (device, precision, N, sign)); fft.cu.
const void* twiddles(int precision, int n, int sign, cudaStream_t st);

}  // namespace gf
