// fft.cu -- batched line FFTs along one axis of a 3D array (stages 2 and 4).
//
// The reference computes its spectra with numpy's pocketfft
// (spectral.forward_dft / inverse_dft, spectral.py:114-130; the landscape's
// inverse, energy.py:343).  Each pass here transforms every line of one axis
// with a mixed-radix Stockham FFT (radix-8 stages, one radix-4/2 stage when
// needed) whose butterflies run in registers: a thread owns 8 points of a
// line per stage, exchanges go through one shared-memory line buffer, the
// first stage reads global memory and the last writes it directly, so each
// pass costs one HBM read and one HBM write of what it touches.
//
// Index bookkeeping of the reference (fftshift / ifftshift / truncation /
// per-axis phase ramps) is folded into the loads and stores:
//   input  element i of a line sits at FFT position
//            i                      (node order, in_centered = 0)
//            (i - Lin/2) mod N      (DC-centred window of Lin modes, zero-padded)
//          times exp(2 pi i m in_phase), m its mode number;
//   output element i reads FFT position
//            i                      (node order)
//            (i - Lout/2) mod N     (DC-centred window of Lout modes: truncation)
//          times scale * exp(2 pi i m out_phase).
// Phases 0 and 1/2 ((-1)^m, the centred-DFT identity) cost nothing.
//
// Tile: one CTA owns B lines; threads (b fastest) so that for strided axes
// the B lines are B consecutive positions of the contiguous axis -- global
// accesses are coalesced for every axis.
#include "../../include/geofield_b200.h"
#include <cuda.h>
#include <cudaTypedefs.h>
#include "common.cuh"
#include "fft_core.cuh"

#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>

namespace gf {
namespace {

struct FftArgs {
  const void* in;
  void* out;
  const void* tw;  // twiddle table W_N^m = exp(sign 2 pi i m / N), m < N
  int shape_in[3];
  int shape_out[3];
  int axis;
  int in_centered, out_centered;
  int sign;
  int in_phase_kind, out_phase_kind;  // 0: none, 1: (-1)^m, 2: general
  double in_phase, out_phase, scale;
};

// One CTA: B lines x (N / 8) threads (N >= 8), b fastest.
template <typename T, int N, int B>
__global__ void __launch_bounds__(B*(N >= 8 ? N / 8 : 1)) fft_kernel(FftArgs a) {
  constexpr int TPL = FftShape<N>::TPL;  // threads per line
  constexpr int PT = FftShape<N>::PT;    // points per thread
  constexpr int LD = LineLD<T, N>::value;  // padded line stride
  extern __shared__ __align__(128) unsigned char fft_smem[];
  cx<T>* buf = reinterpret_cast<cx<T>*>(fft_smem);
  const int tid = threadIdx.x;
  const int ax = a.axis;
  // contiguous axis: lanes walk along a line (coalesced 8-16 B x 32);
  // strided axes: lanes walk across B adjacent lines (B x element >= 128 B)
  const int b = ax == 2 ? tid / TPL : tid % B;
  const int j = ax == 2 ? tid % TPL : tid / B;  // thread index within the line
  const int Lin = a.shape_in[ax], Lout = a.shape_out[ax];
  const cx<T>* __restrict__ in = reinterpret_cast<const cx<T>*>(a.in);
  cx<T>* __restrict__ out = reinterpret_cast<cx<T>*>(a.out);
  const cx<T>* __restrict__ tw = reinterpret_cast<const cx<T>*>(a.tw);

  // ---- line addressing
  int64_t base_in, base_out, st_in, st_out;
  bool live;
  if (ax == 2) {
    const int64_t lines = (int64_t)a.shape_in[0] * a.shape_in[1];
    const int64_t l = (int64_t)blockIdx.x * B + b;
    live = l < lines;
    base_in = l * Lin;
    base_out = l * Lout;
    st_in = 1;
    st_out = 1;
  } else {
    const int s2 = a.shape_in[2];
    const int ptiles = (s2 + B - 1) / B;
    const int o = blockIdx.x / ptiles, p = (blockIdx.x % ptiles) * B + b;
    live = p < s2;
    if (ax == 0) {
      base_in = (int64_t)o * s2 + p;
      base_out = (int64_t)o * a.shape_out[2] + p;
      st_in = (int64_t)a.shape_in[1] * s2;
      st_out = (int64_t)a.shape_out[1] * a.shape_out[2];
    } else {
      base_in = (int64_t)o * a.shape_in[1] * s2 + p;
      base_out = (int64_t)o * a.shape_out[1] * a.shape_out[2] + p;
      st_in = s2;
      st_out = a.shape_out[2];
    }
  }

  // ---- first stage input: positions pos = j + r * (N / PT) of the line
  cx<T> v[PT];
  const int hin = Lin / 2;
#pragma unroll
  for (int r = 0; r < PT; ++r) {
    const int pos = j + r * TPL;
    int src, m;
    if (a.in_centered) {
      m = pos < N / 2 ? pos : pos - N;  // mode at this FFT position
      src = m + hin;
      if (src < 0 || src >= Lin) src = -1;
    } else {
      m = pos;
      src = pos;
    }
    cx<T> x = mk<T>(0, 0);
    if (live && src >= 0) {
      x = in[base_in + (int64_t)src * st_in];
      if (a.in_phase_kind) x = x * phase_factor<T>(a.in_phase_kind, a.in_phase, m);
    }
    v[r] = x;
  }

  // ---- transform (natural-order result in the line buffer)
  cx<T>* line = buf + b * LD;
  fft_line<T, N>(v, line, j, tw, a.sign);

  // ---- output: positions pos = j + r * TPL
  const int hout = Lout / 2;
#pragma unroll
  for (int r = 0; r < PT; ++r) {
    const int pos = j + r * TPL;
    int dst, m;
    if (a.out_centered) {
      m = pos < N / 2 ? pos : pos - N;
      dst = m + hout;
      if (dst < 0 || dst >= Lout) continue;
    } else {
      m = pos;
      dst = pos;
    }
    if (!live) continue;
    cx<T> y = line[sidx<T>(pos)];
    y = mk<T>(y.re * (T)a.scale, y.im * (T)a.scale);
    if (a.out_phase_kind) y = y * phase_factor<T>(a.out_phase_kind, a.out_phase, m);
    out[base_out + (int64_t)dst * st_out] = y;
  }
}

struct LineAddr {
  int64_t base_in, base_out, st_in, st_out;
  bool live;
};

// Addresses of line b of contiguous-axis tile `tile` (B lines per tile).
template <int B>
__device__ __forceinline__ LineAddr line_addr(const FftArgs& a, int64_t tile, int b) {
  LineAddr L;
  const int64_t lines = (int64_t)a.shape_in[0] * a.shape_in[1];
  const int64_t l = tile * B + b;
  L.live = l < lines;
  L.base_in = l * a.shape_in[2];
  L.base_out = l * a.shape_out[2];
  L.st_in = 1;
  L.st_out = 1;
  return L;
}

template <typename T, int N>
__device__ __forceinline__ void store_line(const FftArgs& a, const LineAddr& L, int j, const cx<T>* line) {
  constexpr int TPL = N / 8;
  cx<T>* __restrict__ out = reinterpret_cast<cx<T>*>(a.out);
  const int Lout = a.shape_out[a.axis], hout = Lout / 2;
  if (!L.live) return;
  if (!a.out_centered && !a.out_phase_kind && a.scale == 1.0 && L.st_out == 1) {
    // node-order output of a contiguous line, no scale or phase: a plain copy
    cx<T>* __restrict__ o = out + L.base_out;
#pragma unroll
    for (int r = 0; r < 8; ++r) o[j + r * TPL] = line[sidx<T>(j + r * TPL)];
    return;
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    int dst, m;
    if (a.out_centered) {
      m = pos < N / 2 ? pos : pos - N;
      dst = m + hout;
      if (dst < 0 || dst >= Lout) continue;
    } else {
      m = pos;
      dst = pos;
    }
    cx<T> y = line[sidx<T>(pos)];
    y = mk<T>(y.re * (T)a.scale, y.im * (T)a.scale);
    if (a.out_phase_kind) y = y * phase_factor<T>(a.out_phase_kind, a.out_phase, m);
    out[L.base_out + (int64_t)dst * L.st_out] = y;
  }
}

// Contiguous axis, staged: a persistent CTA streams tiles of B consecutive
// input lines (one contiguous B * Lin block) into shared memory with 1-D
// bulk async copies (cp.async.bulk + mbarrier transaction counts), two
// tiles ahead, so HBM reads run under the butterflies and exchanges without
// holding registers.  Threads then read their first-stage points from the
// staging buffer (unit stride, conflict-free).  Same semantics as fft_kernel.
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  }
}

template <typename T, int N, int B>
__global__ void __launch_bounds__(B * (N / 8)) fft_rows_staged_kernel(FftArgs a, int64_t ntiles) {
  constexpr int TPL = N / 8;
  constexpr int LD = LineLD<T, N>::value;
  extern __shared__ __align__(128) unsigned char fft_smem[];
  const int Lin = a.shape_in[2];
  const int tile_elems = B * Lin;  // multiple of 2 (16-byte granules) -- checked by the launcher
  uint64_t* bars = reinterpret_cast<uint64_t*>(fft_smem);
  cx<T>* stage0 = reinterpret_cast<cx<T>*>(fft_smem + 128);
  cx<T>* lines = stage0 + 2 * tile_elems;
  const int tid = threadIdx.x;
  const int b = tid / TPL, j = tid % TPL;
  const int64_t nlines = (int64_t)a.shape_in[0] * a.shape_in[1];
  const cx<T>* __restrict__ in = reinterpret_cast<const cx<T>*>(a.in);
  const cx<T>* __restrict__ tw = reinterpret_cast<const cx<T>*>(a.tw);
  auto issue = [&](int64_t t, int s) {
    const int64_t l0 = t * B;
    const int64_t nl = nlines - l0 < B ? nlines - l0 : B;
    bulk_load(stage0 + s * tile_elems, in + l0 * Lin, (unsigned)(nl * Lin * sizeof(cx<T>)), &bars[s]);
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    if (blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  cx<T>* line = lines + b * LD;
  const int hin = Lin / 2;
  // this thread's source positions in its line (the same for every tile), -1: zero
  int spos[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    if (a.in_centered) {
      const int m = pos < N / 2 ? pos : pos - N;
      spos[r] = (m + hin < 0 || m + hin >= Lin) ? -1 : m + hin;
    } else {
      spos[r] = pos < Lin ? pos : -1;
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it & 1;
    mbar_wait(&bars[s], (it >> 1) & 1);
    const LineAddr L = line_addr<B>(a, tile, b);
    const cx<T>* src_line = stage0 + s * tile_elems + b * Lin;
    cx<T> v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = (L.live && spos[r] >= 0) ? src_line[spos[r]] : mk<T>(0, 0);
    if (a.in_phase_kind) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int pos = j + r * TPL;
        const int m = a.in_centered ? (pos < N / 2 ? pos : pos - N) : pos;
        if (L.live && spos[r] >= 0) v[r] = v[r] * phase_factor<T>(a.in_phase_kind, a.in_phase, m);
      }
    }
    __syncthreads();  // stage s fully read: refill it two tiles ahead
    if (tid == 0 && tile + 2 * gridDim.x < ntiles) issue(tile + 2 * gridDim.x, s);
    fft_line<T, N>(v, line, j, tw, a.sign);
    store_line<T, N>(a, L, j, line);
  }
}

// Strided axes, TMA-staged: a persistent CTA owns tiles of RB lines (RB
// consecutive positions of the contiguous axis = one 128-byte row per line
// position).  Tiles arrive by tensor-map bulk copies (3-D boxes of <= 256
// rows) into a [row][RB] shared tile, three buffers deep, two tiles ahead;
// the FFT runs in place in that tile (lanes walk the RB columns: every
// exchange is a full conflict-free row); the result leaves by tensor-map
// bulk stores.  No register staging of HBM traffic, no LSU instructions for
// it -- the issue slots go to the butterflies.  Same semantics as fft_kernel.
struct TmaGeom {
  int rin, nbin;          // input box rows, boxes per tile
  int rout;               // output box rows
  int ptiles;             // tiles along the contiguous axis
};

__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* tm, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
               "r"(c0), "r"(c1), "r"(c2), "r"((unsigned)__cvta_generic_to_shared(src))
               : "memory");
}

template <typename T, int N>
__global__ void __launch_bounds__((128 / sizeof(cx<T>)) * (N / 8))
    fft_cols_tma_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, FftArgs a,
                        TmaGeom g, int64_t ntiles) {
  constexpr int RB = 128 / sizeof(cx<T>);  // lines per tile (one 128-byte row)
  constexpr int TPL = N / 8;
  constexpr int U = sizeof(cx<T>) / 8;     // 8-byte tensor-map units per element
  extern __shared__ __align__(128) unsigned char fft_smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(fft_smem);
  cx<T>* bufs = reinterpret_cast<cx<T>*>(fft_smem + 128);
  const int tid = threadIdx.x;
  const int b = tid % RB, j = tid / RB;
  const int ax = a.axis;
  const int Lin = a.shape_in[ax], Lout = a.shape_out[ax], hin = Lin / 2, hout = Lout / 2;
  const cx<T>* __restrict__ tw = reinterpret_cast<const cx<T>*>(a.tw);
  const unsigned tx_bytes = (unsigned)(g.nbin * g.rin * 128);
  auto coords = [&](int64_t t, int row, int& c0, int& c1, int& c2) {
    const int o = (int)(t / g.ptiles), p0 = (int)(t % g.ptiles) * RB;
    c0 = p0 * U;
    if (ax == 1) {
      c1 = row;
      c2 = o;
    } else {
      c1 = o;
      c2 = row;
    }
  };
  auto issue_load = [&](int64_t t, int s) {
    cx<T>* dst = bufs + (size_t)s * N * RB;
    const unsigned bb = (unsigned)__cvta_generic_to_shared(&bars[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(tx_bytes) : "memory");
    for (int k = 0; k < g.nbin; ++k) {
      int c0, c1, c2;
      coords(t, k * g.rin, c0, c1, c2);
      tma_load3(dst + (size_t)k * g.rin * RB, &tin, c0, c1, c2, &bars[s]);
    }
  };
  if (tid == 0) {
    for (int s = 0; s < 3; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (blockIdx.x < ntiles) issue_load(blockIdx.x, 0);
    if (blockIdx.x + gridDim.x < ntiles) issue_load(blockIdx.x + gridDim.x, 1);
  }
  __syncthreads();
  // this thread's input rows (the same for every tile): source row or -1
  int srow[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    if (a.in_centered) {
      const int m = pos < N / 2 ? pos : pos - N;
      srow[r] = (m + hin < 0 || m + hin >= Lin) ? -1 : (m + hin) * RB + b;
    } else {
      srow[r] = pos * RB + b;
    }
  }
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int s = it % 3;
    cx<T>* buf = bufs + (size_t)s * N * RB;
    mbar_wait(&bars[s], (it / 3) & 1);
    cx<T> v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = srow[r] >= 0 ? buf[srow[r]] : mk<T>(0, 0);
    if (a.in_phase_kind) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int pos = j + r * TPL;
        const int m = a.in_centered ? (pos < N / 2 ? pos : pos - N) : pos;
        if (srow[r] >= 0) v[r] = v[r] * phase_factor<T>(a.in_phase_kind, a.in_phase, m);
      }
    }
    if (a.scale != 1.0 && !a.out_phase_kind) {  // linear: scale the inputs, no extra pass over the tile
      const T sc = (T)a.scale;
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = mk<T>(v[r].re * sc, v[r].im * sc);
    }
    fft_line<T, N, RB>(v, buf + b, j, tw, a.sign);  // ends with __syncthreads
    if (a.out_phase_kind) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int pos = j + r * TPL;
        const int m = a.out_centered ? (pos < N / 2 ? pos : pos - N) : pos;
        cx<T> y = buf[pos * RB + b];
        y = mk<T>(y.re * (T)a.scale, y.im * (T)a.scale);
        if (a.out_phase_kind) y = y * phase_factor<T>(a.out_phase_kind, a.out_phase, m);
        buf[pos * RB + b] = y;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      // output rows: node order -> rows [0, N); centred -> dst [0, hout) from
      // pos [N - hout, N) and dst [hout, Lout) from pos [0, Lout - hout)
      int c0, c1, c2;
      if (!a.out_centered) {
        for (int r0 = 0; r0 < N; r0 += g.rout) {
          coords(tile, r0, c0, c1, c2);
          tma_store3(&tout, c0, c1, c2, buf + (size_t)r0 * RB);
        }
      } else {
        for (int r0 = 0; r0 < hout; r0 += g.rout) {
          coords(tile, r0, c0, c1, c2);
          tma_store3(&tout, c0, c1, c2, buf + (size_t)(N - hout + r0) * RB);
        }
        for (int r0 = hout; r0 < Lout; r0 += g.rout) {
          coords(tile, r0, c0, c1, c2);
          tma_store3(&tout, c0, c1, c2, buf + (size_t)(r0 - hout) * RB);
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      // the buffer two tiles ahead held the previous tile: its store must
      // have finished reading before the refill
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const int64_t t2 = tile + 2 * (int64_t)gridDim.x;
      if (t2 < ntiles) issue_load(t2, (it + 2) % 3);
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Strided axes, complex64: one thread owns the same FFT positions of two
// adjacent lines (b, b + 1), so every global access is a 16-byte vector and
// half as many load/store instructions feed the LSU (the ncu stall of the
// 8-byte version was lg_throttle).  Same semantics as fft_kernel; requires an
// even contiguous extent (the lines of a pair are both live or both dead).
template <int N, int B>
__global__ void __launch_bounds__(B / 2 * (N / 8), 2) fft_pair_kernel(FftArgs a) {
  using T = float;
  constexpr int TPL = N / 8;
  constexpr int LD = LineLD<T, N>::value;
  constexpr int BP = B / 2;
  extern __shared__ __align__(128) unsigned char fft_smem[];
  cx<T>* buf = reinterpret_cast<cx<T>*>(fft_smem);
  const int tid = threadIdx.x;
  const int ax = a.axis;
  const int bp = tid % BP, j = tid / BP;
  const int Lin = a.shape_in[ax], Lout = a.shape_out[ax];
  const float4* __restrict__ in = reinterpret_cast<const float4*>(a.in);
  float4* __restrict__ out = reinterpret_cast<float4*>(a.out);
  const cx<T>* __restrict__ tw = reinterpret_cast<const cx<T>*>(a.tw);
  const int s2 = a.shape_in[2];
  const int ptiles = (s2 + B - 1) / B;
  const int o = blockIdx.x / ptiles, p = (blockIdx.x % ptiles) * B + 2 * bp;
  const bool live = p < s2;
  int64_t base_in, base_out, st_in, st_out;  // in float4 (pair) units
  if (ax == 0) {
    base_in = ((int64_t)o * s2 + p) / 2;
    base_out = ((int64_t)o * a.shape_out[2] + p) / 2;
    st_in = (int64_t)a.shape_in[1] * s2 / 2;
    st_out = (int64_t)a.shape_out[1] * a.shape_out[2] / 2;
  } else {
    base_in = ((int64_t)o * a.shape_in[1] * s2 + p) / 2;
    base_out = ((int64_t)o * a.shape_out[1] * a.shape_out[2] + p) / 2;
    st_in = s2 / 2;
    st_out = a.shape_out[2] / 2;
  }
  cx<T> v0[8], v1[8];
  const int hin = Lin / 2;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    int src, m;
    if (a.in_centered) {
      m = pos < N / 2 ? pos : pos - N;
      src = m + hin;
      if (src < 0 || src >= Lin) src = -1;
    } else {
      m = pos;
      src = pos;
    }
    cx<T> x0 = mk<T>(0, 0), x1 = mk<T>(0, 0);
    if (live && src >= 0) {
      const float4 q = __ldcs(&in[base_in + (int64_t)src * st_in]);
      x0 = mk<T>(q.x, q.y);
      x1 = mk<T>(q.z, q.w);
      if (a.in_phase_kind) {
        const cx<T> ph = phase_factor<T>(a.in_phase_kind, a.in_phase, m);
        x0 = x0 * ph;
        x1 = x1 * ph;
      }
    }
    v0[r] = x0;
    v1[r] = x1;
  }
  cx<T>* line0 = buf + (2 * bp) * LD;
  cx<T>* line1 = line0 + LD;
  // park line 1 in its own (so far untouched) buffer while line 0 transforms
#pragma unroll
  for (int r = 0; r < 8; ++r) line1[sidx<T>(j + r * TPL)] = v1[r];
  fft_line<T, N>(v0, line0, j, tw, a.sign);
#pragma unroll
  for (int r = 0; r < 8; ++r) v1[r] = line1[sidx<T>(j + r * TPL)];
  fft_line<T, N>(v1, line1, j, tw, a.sign);
  if (!live) return;
  const int hout = Lout / 2;
  const T sc = (T)a.scale;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    int dst, m;
    if (a.out_centered) {
      m = pos < N / 2 ? pos : pos - N;
      dst = m + hout;
      if (dst < 0 || dst >= Lout) continue;
    } else {
      m = pos;
      dst = pos;
    }
    cx<T> y0 = line0[sidx<T>(pos)], y1 = line1[sidx<T>(pos)];
    y0 = mk<T>(y0.re * sc, y0.im * sc);
    y1 = mk<T>(y1.re * sc, y1.im * sc);
    if (a.out_phase_kind) {
      const cx<T> ph = phase_factor<T>(a.out_phase_kind, a.out_phase, m);
      y0 = y0 * ph;
      y1 = y1 * ph;
    }
    __stcs(&out[base_out + (int64_t)dst * st_out], make_float4(y0.re, y0.im, y1.re, y1.im));
  }
}

// Strided y pass fused with the slab exchange of the multi-GPU landscape
// (parallel.score_field_slab): the transformed lines are stored straight into
// the destination rank's y-slab -- a peer GPU's buffer over NVLink when the
// pointer is a peer mapping -- instead of a local buffer followed by an
// all-to-all.  Element (x, y, z) of this rank's planes lands in rank s with
// ybound[s] <= y < ybound[s+1] at ((x_off + x) * ny_s + y - ybound[s]) * N2 + z.
// Loads, butterflies and scaling are those of fft_kernel (bitwise the same
// values); lanes walk 16 (8) adjacent z, so every store is a 128-byte row.
constexpr int kMaxScatter = 8;
struct ScatterOut {
  int nranks;
  int ybound[kMaxScatter + 1];
  void* dst[kMaxScatter];
  int x_off;
};

template <typename T, int N, int B>
__global__ void __launch_bounds__(B * (N / 8)) fft_scatter_kernel(FftArgs a, ScatterOut so) {
  constexpr int TPL = N / 8;
  constexpr int LD = LineLD<T, N>::value;
  extern __shared__ __align__(128) unsigned char fft_smem[];
  cx<T>* buf = reinterpret_cast<cx<T>*>(fft_smem);
  const int tid = threadIdx.x;
  const int b = tid % B, j = tid / B;
  const int Lin = a.shape_in[1], s2 = a.shape_in[2];
  const int ptiles = (s2 + B - 1) / B;
  const int o = blockIdx.x / ptiles, p = (blockIdx.x % ptiles) * B + b;
  const bool live = p < s2;
  const cx<T>* __restrict__ in = reinterpret_cast<const cx<T>*>(a.in);
  const cx<T>* __restrict__ tw = reinterpret_cast<const cx<T>*>(a.tw);
  const int64_t base_in = (int64_t)o * Lin * s2 + p;
  const int hin = Lin / 2;
  cx<T> v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    int src, m;
    if (a.in_centered) {
      m = pos < N / 2 ? pos : pos - N;
      src = m + hin;
      if (src < 0 || src >= Lin) src = -1;
    } else {
      m = pos;
      src = pos;
    }
    cx<T> x = mk<T>(0, 0);
    if (live && src >= 0) {
      x = in[base_in + (int64_t)src * s2];
      if (a.in_phase_kind) x = x * phase_factor<T>(a.in_phase_kind, a.in_phase, m);
    }
    v[r] = x;
  }
  cx<T>* line = buf + b * LD;
  fft_line<T, N>(v, line, j, tw, a.sign);
  if (!live) return;
  const int Lout = a.shape_out[1], hout = Lout / 2;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int pos = j + r * TPL;
    int y, m;  // output row and mode number of FFT position pos
    if (a.out_centered) {
      m = pos < N / 2 ? pos : pos - N;
      y = m + hout;
      if (y < 0 || y >= Lout) continue;  // truncated away
    } else {
      m = pos;
      y = pos;
    }
    int s = 0;
    while (s + 1 < so.nranks && y >= so.ybound[s + 1]) ++s;
    const int ny = so.ybound[s + 1] - so.ybound[s];
    cx<T> val = line[sidx<T>(pos)];
    val = mk<T>(val.re * (T)a.scale, val.im * (T)a.scale);
    if (a.out_phase_kind) val = val * phase_factor<T>(a.out_phase_kind, a.out_phase, m);
    cx<T>* dst = reinterpret_cast<cx<T>*>(so.dst[s]);
    dst[((int64_t)(so.x_off + o) * ny + (y - so.ybound[s])) * s2 + p] = val;
  }
}

template <typename T, int N>
cudaError_t launch_scatter_n(const FftArgs& a, const ScatterOut& so, cudaStream_t st) {
  constexpr int TPL = N / 8;
  constexpr int B0 = 128 / sizeof(cx<T>);
  constexpr int B = B0 * TPL > 1024 ? 1024 / TPL : B0;
  constexpr size_t smem = sizeof(cx<T>) * B * LineLD<T, N>::value;
  {
    cudaError_t e = ensure_smem((const void*)fft_scatter_kernel<T, N, B>, smem);
    if (e != cudaSuccess) return e;
  }
  const int64_t blocks = (int64_t)a.shape_in[0] * ceil_div(a.shape_in[2], B);
  fft_scatter_kernel<T, N, B><<<(unsigned)blocks, B * TPL, smem, st>>>(a, so);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_scatter(const FftArgs& a, const ScatterOut& so, int n, cudaStream_t st) {
  switch (n) {
    case 8: return launch_scatter_n<T, 8>(a, so, st);
    case 16: return launch_scatter_n<T, 16>(a, so, st);
    case 32: return launch_scatter_n<T, 32>(a, so, st);
    case 64: return launch_scatter_n<T, 64>(a, so, st);
    case 128: return launch_scatter_n<T, 128>(a, so, st);
    case 256: return launch_scatter_n<T, 256>(a, so, st);
    case 512: return launch_scatter_n<T, 512>(a, so, st);
    case 1024: return launch_scatter_n<T, 1024>(a, so, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename T>
__global__ void twiddle_kernel(cx<T>* tw, int n, int sign) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < n; m += gridDim.x * blockDim.x) {
    double s, c;
    sincospi((double)sign * 2.0 * (double)m / (double)n, &s, &c);
    tw[m] = mk<T>((T)c, (T)s);
  }
}

std::mutex g_tw_mu;
std::map<std::tuple<int, int, int, int>, void*> g_tw;  // (device, precision, n, sign) -> table

}  // namespace

const void* twiddles(int precision, int n, int sign, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_tuple(dev, precision, n, sign);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  void* p = nullptr;
  size_t bytes = (size_t)n * (precision == 64 ? 16 : 8);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  if (precision == 64) twiddle_kernel<double><<<(n + 255) / 256, 256, 0, st>>>((cx<double>*)p, n, sign);
  else twiddle_kernel<float><<<(n + 255) / 256, 256, 0, st>>>((cx<float>*)p, n, sign);
  cudaStreamSynchronize(st);
  g_tw[key] = p;
  return p;
}

namespace {

template <typename T, int N, int B>
cudaError_t launch_nb(const FftArgs& a, cudaStream_t st) {
  constexpr int TPL = N >= 8 ? N / 8 : 1;
  int64_t blocks;
  if (a.axis == 2) blocks = ceil_div((int64_t)a.shape_in[0] * a.shape_in[1], B);
  else {
    const int so = a.axis == 0 ? a.shape_in[1] : a.shape_in[0];
    blocks = (int64_t)so * ceil_div(a.shape_in[2], B);
  }
  constexpr size_t smem = sizeof(cx<T>) * B * LineLD<T, N>::value;
  {
    cudaError_t e = ensure_smem((const void*)fft_kernel<T, N, B>, smem);
    if (e != cudaSuccess) return e;
  }
  fft_kernel<T, N, B><<<(unsigned)blocks, B * TPL, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N, int B>
cudaError_t launch_pair(const FftArgs& a, cudaStream_t st) {
  const int so = a.axis == 0 ? a.shape_in[1] : a.shape_in[0];
  const int64_t blocks = (int64_t)so * ceil_div(a.shape_in[2], B);
  constexpr size_t smem = sizeof(cx<float>) * B * LineLD<float, N>::value;
  {
    cudaError_t e = ensure_smem((const void*)fft_pair_kernel<N, B>, smem);
    if (e != cudaSuccess) return e;
  }
  fft_pair_kernel<N, B><<<(unsigned)blocks, B / 2 * (N / 8), smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int N, int B>
cudaError_t launch_staged(const FftArgs& a, cudaStream_t st) {
  const int64_t ntiles = ceil_div((int64_t)a.shape_in[0] * a.shape_in[1], B);
  const size_t smem = 128 + sizeof(cx<T>) * ((size_t)2 * B * a.shape_in[2] + (size_t)B * LineLD<T, N>::value);
  if (smem > 200 * 1024) return launch_nb<T, N, B>(a, st);
  const void* fn = (const void*)fft_rows_staged_kernel<T, N, B>;
  cudaError_t e = ensure_smem(fn, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = resident_ctas(fn, B * (N / 8), smem);
  const int sms = sm_count();
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
  fft_rows_staged_kernel<T, N, B><<<(unsigned)grid, B * (N / 8), smem, st>>>(a, ntiles);
  return cudaGetLastError();
}


PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// 3-D map over a (s0, s1, s2) complex array in 8-byte units; box of 128 bytes
// along s2 and `rows` along the transform axis.
bool encode_map(CUtensorMap* m, const void* base, const int* shape, int esz, int axis, int rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int u = esz / 8;
  cuuint64_t dims[3] = {(cuuint64_t)shape[2] * u, (cuuint64_t)shape[1], (cuuint64_t)shape[0]};
  cuuint64_t strides[2] = {(cuuint64_t)shape[2] * esz, (cuuint64_t)shape[1] * shape[2] * esz};
  cuuint32_t box[3] = {16, axis == 1 ? (cuuint32_t)rows : 1u, axis == 0 ? (cuuint32_t)rows : 1u};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_INT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// returns cudaErrorNotSupported when the shape does not fit the TMA path
template <typename T, int N>
cudaError_t launch_tma(const FftArgs& a, cudaStream_t st) {
  constexpr int RB = 128 / sizeof(cx<T>);
  const int esz = sizeof(cx<T>);
  const int Lin = a.shape_in[a.axis], Lout = a.shape_out[a.axis];
  if (((uintptr_t)a.in & 15) || ((uintptr_t)a.out & 15)) return cudaErrorNotSupported;
  if (((int64_t)a.shape_in[2] * esz) % 16 || ((int64_t)a.shape_out[2] * esz) % 16) return cudaErrorNotSupported;
  if (a.out_centered && (Lout % 2)) return cudaErrorNotSupported;
  TmaGeom g;
  g.rin = Lin < 256 ? Lin : 256;
  g.nbin = (Lin + g.rin - 1) / g.rin;
  if (g.nbin * g.rin > N) return cudaErrorNotSupported;
  g.rout = a.out_centered ? (Lout / 2 < 256 ? Lout / 2 : 256) : (N < 256 ? N : 256);
  if (a.out_centered && (Lout / 2) % g.rout) return cudaErrorNotSupported;
  g.ptiles = (a.shape_in[2] + RB - 1) / RB;
  CUtensorMap tin, tout;
  if (!encode_map(&tin, a.in, a.shape_in, esz, a.axis, g.rin)) return cudaErrorNotSupported;
  if (!encode_map(&tout, a.out, a.shape_out, esz, a.axis, g.rout)) return cudaErrorNotSupported;
  const int so = a.axis == 0 ? a.shape_in[1] : a.shape_in[0];
  const int64_t ntiles = (int64_t)so * g.ptiles;
  const size_t smem = 128 + (size_t)3 * N * 128;
  const void* fn = (const void*)fft_cols_tma_kernel<T, N>;
  cudaError_t e = ensure_smem(fn, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = resident_ctas(fn, RB * (N / 8), smem);
  const int sms = sm_count();
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
  fft_cols_tma_kernel<T, N><<<(unsigned)grid, RB * (N / 8), smem, st>>>(tin, tout, a, g, ntiles);
  return cudaGetLastError();
}

// lines per CTA: strided axes need >= 128 contiguous bytes per row per CTA
// (B = 16 complex64 / 8 complex128) for full-sector, full-line coalescing;
// the contiguous axis only needs enough threads (B * N / 8 >= 256).
template <typename T, int N>
cudaError_t launch_n(const FftArgs& a, cudaStream_t st) {
  constexpr int TPL = N >= 8 ? N / 8 : 1;
  constexpr int B_row = 128 / sizeof(cx<T>);
  constexpr int B_thr = (256 / TPL) < 1 ? 1 : (256 / TPL) > 32 ? 32 : (256 / TPL);
  constexpr int B_str = (B_row > B_thr ? B_row : B_thr) * TPL > 1024 ? 1024 / TPL : (B_row > B_thr ? B_row : B_thr);
  if constexpr (N >= 64) {
    if (a.axis == 2 && ((int64_t)B_thr * a.shape_in[2] * sizeof(cx<T>)) % 16 == 0 &&
        ((uintptr_t)a.in & 15) == 0)
      return launch_staged<T, N, B_thr>(a, st);
  }
  if (a.axis == 2) return launch_nb<T, N, B_thr>(a, st);
  if constexpr (N >= 64 && N <= 512) {
    cudaError_t e = launch_tma<T, N>(a, st);
    if (e != cudaErrorNotSupported) return e;
  }
  if constexpr (sizeof(T) == 4 && N >= 64 && N <= 512) {
    if (a.shape_in[2] % 2 == 0 && a.shape_out[2] % 2 == 0) return launch_pair<N, 16>(a, st);
  }
  return launch_nb<T, N, B_str>(a, st);
}

template <typename T>
cudaError_t launch_fft(const FftArgs& a, int n, cudaStream_t st) {
  switch (n) {
    case 2: return launch_n<T, 2>(a, st);
    case 4: return launch_n<T, 4>(a, st);
    case 8: return launch_n<T, 8>(a, st);
    case 16: return launch_n<T, 16>(a, st);
    case 32: return launch_n<T, 32>(a, st);
    case 64: return launch_n<T, 64>(a, st);
    case 128: return launch_n<T, 128>(a, st);
    case 256: return launch_n<T, 256>(a, st);
    case 512: return launch_n<T, 512>(a, st);
    case 1024: return launch_n<T, 1024>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

int phase_kind(double ph) {
  double f = ph - floor(ph);
  if (f == 0.0) return 0;
  if (f == 0.5) return 1;
  return 2;
}

}  // namespace
}  // namespace gf

using namespace gf;

extern "C" int gf_fft_pass(int precision, const void* in, void* out, const int32_t* shape_in,
                           const int32_t* shape_out, int axis, int n, int in_centered, int out_centered, int sign,
                           double in_phase, double out_phase, double scale, void* stream) {
  GF_CHECK(in && out && shape_in && shape_out, GF_EINVAL, "null argument");
  GF_CHECK(axis >= 0 && axis < 3, GF_EINVAL, "axis must be 0, 1 or 2");
  GF_CHECK(n >= 2 && n <= 1024 && (n & (n - 1)) == 0, GF_EINVAL, "FFT length must be a power of two in [2, 1024]");
  GF_CHECK(sign == -1 || sign == 1, GF_EINVAL, "sign must be -1 or +1");
  GF_CHECK(precision == 32 || precision == 64, GF_EINVAL, "precision must be 32 or 64");
  for (int a = 0; a < 3; ++a)
    if (a != axis) GF_CHECK(shape_in[a] == shape_out[a], GF_EINVAL, "non-transform axes must match");
  GF_CHECK(shape_in[axis] <= n && shape_out[axis] <= n, GF_EINVAL, "line longer than the FFT length");
  GF_CHECK(in_centered || shape_in[axis] == n, GF_EINVAL, "node-ordered input must have length n");
  GF_CHECK(out_centered || shape_out[axis] == n, GF_EINVAL, "node-ordered output must have length n");
  cudaStream_t st = (cudaStream_t)stream;
  FftArgs a = {};
  a.in = in;
  a.out = out;
  a.tw = twiddles(precision, n, sign, st);
  GF_CHECK(a.tw != nullptr, GF_ENOMEM, "twiddle table allocation failed");
  for (int k = 0; k < 3; ++k) {
    a.shape_in[k] = shape_in[k];
    a.shape_out[k] = shape_out[k];
  }
  a.axis = axis;
  a.in_centered = in_centered;
  a.out_centered = out_centered;
  a.sign = sign;
  a.in_phase = in_phase;
  a.out_phase = out_phase;
  a.in_phase_kind = phase_kind(in_phase);
  a.out_phase_kind = phase_kind(out_phase);
  a.scale = scale;
  if (precision == 64) GF_CUDA(launch_fft<double>(a, n, st));
  else GF_CUDA(launch_fft<float>(a, n, st));
  return 0;
}

extern "C" int gf_fft_pass_scatter(int precision, const void* in, const int32_t* shape_in, int n, int in_centered,
                                   int out_len, int out_centered, int sign, double in_phase, double out_phase,
                                   double scale, int nranks, const int32_t* y_bounds, const uint64_t* dst_ptrs,
                                   int x_off, void* stream) {
  GF_CHECK(in && shape_in && y_bounds && dst_ptrs, GF_EINVAL, "null argument");
  GF_CHECK(nranks >= 1 && nranks <= kMaxScatter, GF_EINVAL, "1 to 8 destination ranks");
  GF_CHECK(n >= 8 && n <= 1024 && (n & (n - 1)) == 0, GF_EINVAL, "FFT length must be a power of two in [8, 1024]");
  GF_CHECK(precision == 32 || precision == 64, GF_EINVAL, "precision must be 32 or 64");
  GF_CHECK(sign == -1 || sign == 1, GF_EINVAL, "sign must be -1 or +1");
  GF_CHECK(shape_in[1] <= n && (in_centered || shape_in[1] == n), GF_EINVAL, "bad line length");
  GF_CHECK(out_len <= n && (out_centered || out_len == n), GF_EINVAL, "bad output length");
  GF_CHECK(y_bounds[0] == 0 && y_bounds[nranks] == out_len, GF_EINVAL, "y slabs must tile the output rows");
  for (int r = 0; r < nranks; ++r) {
    GF_CHECK(y_bounds[r + 1] >= y_bounds[r], GF_EINVAL, "y slab bounds must be non-decreasing");
    GF_CHECK(dst_ptrs[r] != 0 || y_bounds[r + 1] == y_bounds[r], GF_EINVAL, "null destination slab");
  }
  GF_CHECK(x_off >= 0, GF_EINVAL, "negative plane offset");
  cudaStream_t st = (cudaStream_t)stream;
  FftArgs a = {};
  a.in = in;
  a.out = nullptr;
  a.tw = twiddles(precision, n, sign, st);
  GF_CHECK(a.tw != nullptr, GF_ENOMEM, "twiddle table allocation failed");
  for (int k = 0; k < 3; ++k) a.shape_in[k] = shape_in[k];
  a.shape_out[0] = shape_in[0];
  a.shape_out[1] = out_len;
  a.shape_out[2] = shape_in[2];
  a.axis = 1;
  a.in_centered = in_centered;
  a.out_centered = out_centered;
  a.sign = sign;
  a.in_phase = in_phase;
  a.in_phase_kind = phase_kind(in_phase);
  a.out_phase = out_phase;
  a.out_phase_kind = phase_kind(out_phase);
  a.scale = scale;
  ScatterOut so = {};
  so.nranks = nranks;
  for (int r = 0; r <= nranks; ++r) so.ybound[r] = y_bounds[r];
  for (int r = 0; r < nranks; ++r) so.dst[r] = reinterpret_cast<void*>(dst_ptrs[r]);
  so.x_off = x_off;
  if (shape_in[0] == 0) return 0;
  if (precision == 64) GF_CUDA(launch_scatter<double>(a, so, n, st));
  else GF_CUDA(launch_scatter<float>(a, so, n, st));
  return 0;
}
