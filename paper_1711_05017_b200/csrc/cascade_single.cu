// cascade_single.cu -- latency kernel for ONE pose (the haptic query, Q1).
//
// Same semantics as cascade.cu (reference _core.cascade_3d,
// /root/reference/pkg/src/geofield/_core.pyx:598-724).  A lone query has
// only ~10^5-10^6 modes, so latency is set by how many warps are resident
// and how long each thread's dependency chain is, not by bandwidth:
//   * every thread handles ~1-3 modes (no per-run setup): the translation
//     phase comes from per-axis tables px/py/pz built once per CTA
//     (sincospi of float64-reduced arguments), the continuous index from 9
//     FMAs, so no thread waits on a long serial chain;
//   * register cap 64 (4 CTAs of 256 threads per SM, 32 warps) so the grid
//     is one resident wave of 4 x 148 CTAs that hides gather latency;
//   * the 26 moments are reduced through a shared-memory transpose (fixed
//     order) instead of 26 five-level shuffle trees, then across CTAs by a
//     last-block-done pass in fixed block order (bitwise repeatable).
// Lane layout: the same per-pose oriented 4 x 8 patches as cascade.cu, so
// the corner gathers of a warp share few 128-byte lines.
#include "cascade.cuh"
#include "common.cuh"

#include <math.h>
#include <stdlib.h>

namespace gf {
namespace {

constexpr int kThreads = 256;

struct SinglePose {
  double mu[3][3];
  double R[9];
  double targ[3];
  int p, q, r, nP, nQ;
};

__device__ __forceinline__ double exact_u_s(const double* R, const double* dom, int a, int kx, int ky, int kz,
                                            int hx, int hy, int hz, int ha) {
  double ox = __dmul_rn((double)(kx - hx), dom[0]);
  double oy = __dmul_rn((double)(ky - hy), dom[1]);
  double oz = __dmul_rn((double)(kz - hz), dom[2]);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(R[0 + a], ox), __dmul_rn(R[3 + a], oy)), __dmul_rn(R[6 + a], oz));
  return __dadd_rn(__ddiv_rn(-s, dom[a]), (double)ha);
}

// Output slot i (0..13, interleaved complex) as a linear form of the 26
// moments; called by 14 threads in parallel.
__device__ __forceinline__ double finalize_slot(const CascadeArgs& a, const double* R, const double* m, int i) {
  const double TWO_PI = 6.283185307179586;
  const double dc = a.dcell;
  if (i < 2) return dc * m[i];
  if (i < 8) {  // T_a = 2 pi i dw_a Z_a
    int ax = (i - 2) >> 1;
    double k = dc * TWO_PI * a.dom[ax];
    return (i & 1) ? k * m[2 + 2 * ax] : -k * m[3 + 2 * ax];
  }
  const int g = (i - 8) >> 1, im = i & 1;
  // A_g = Omega_g R: rows (generator g) -- see _core.pyx:615-626
  double A[3][3];
  for (int b = 0; b < 3; ++b) {
    double r0 = R[b], r1 = R[3 + b], r2 = R[6 + b];
    if (g == 0) { A[0][b] = 0.0; A[1][b] = -r2; A[2][b] = r1; }
    else if (g == 1) { A[0][b] = r2; A[1][b] = 0.0; A[2][b] = -r0; }
    else { A[0][b] = -r1; A[1][b] = r0; A[2][b] = 0.0; }
  }
  double acc = 0.0;
  for (int b = 0; b < 3; ++b)
    for (int ax = 0; ax < 3; ++ax) acc += -A[ax][b] * (a.dom[ax] / a.dom[b]) * m[8 + im + 2 * (3 * b + ax)];
  for (int ax = 0; ax < 3; ++ax) {
    double q = A[ax][0] * a.center[0] + A[ax][1] * a.center[1] + A[ax][2] * a.center[2];
    double k = TWO_PI * a.dom[ax] * q;
    acc += im ? k * m[2 + 2 * ax] : -k * m[3 + 2 * ax];
  }
  return dc * acc;
}

template <typename T, bool WRAP>
__global__ void __launch_bounds__(kThreads, (sizeof(T) == 4 ? 3 : 2)) cascade3d_single_kernel(CascadeArgs a) {
  using P4 = typename pair4<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // dynamic: transpose buffer tr[26][257] (reduction) | px | py | pz
  T(*tr)[kThreads + 1] = reinterpret_cast<T(*)[kThreads + 1]>(smem_raw);
  cx<T>* ptab = reinterpret_cast<cx<T>*>(smem_raw + sizeof(T) * kNumMoments * (kThreads + 1) + 16);
  __shared__ SinglePose sp;
  __shared__ double red[kNumMoments];
  __shared__ unsigned ticket;

  const int tid = threadIdx.x;
  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  const double* src = a.poses ? a.poses + a.pose_offset * 12 : a.pose_inline;
  if (tid < 9) {
    sp.R[tid] = src[tid];
    int ia = tid / 3, ib = tid % 3;
    sp.mu[ia][ib] = -src[ib * 3 + ia] * (a.dom[ib] / a.dom[ia]);
  }
  if (tid >= 16 && tid < 19) sp.targ[tid - 16] = a.dom[tid - 16] * src[9 + tid - 16];
  __syncthreads();
  if (tid == 0) {
    int r = 2;
    if (a.dim == 3) {
      double z0 = fabs(sp.mu[2][0]), z1 = fabs(sp.mu[2][1]), z2 = fabs(sp.mu[2][2]);
      r = (z0 <= z1 && z0 <= z2) ? 0 : (z1 <= z2 ? 1 : 2);
    }
    int o1 = (r + 1) % 3, o2 = (r + 2) % 3;
    if (a.dim == 2) { o1 = 0; o2 = 1; }
    bool sw = fabs(sp.mu[2][o1]) > fabs(sp.mu[2][o2]);
    sp.p = sw ? o2 : o1;
    sp.q = sw ? o1 : o2;
    sp.r = r;
    sp.nP = ((sp.p == 0 ? w0 : (sp.p == 1 ? w1 : w2)) + 15) / 16;
    sp.nQ = ((sp.q == 0 ? w0 : (sp.q == 1 ? w1 : w2)) + 15) / 16;
  }
  for (int i = tid; i < w0 + w1 + w2; i += kThreads) {
    int ax = i < w0 ? 0 : (i < w0 + w1 ? 1 : 2);
    int k = i - (ax == 0 ? 0 : (ax == 1 ? w0 : w0 + w1));
    int hh = ax == 0 ? hx : (ax == 1 ? hy : hz);
    double cyc = sp.targ[ax] * (double)(k - hh);
    cyc -= rint(cyc);
    T sn, cs;
    if constexpr (sizeof(T) == 4) sincospif(2.0f * (float)cyc, &sn, &cs);
    else sincospi(2.0 * cyc, &sn, &cs);
    ptab[i] = mk<T>(cs, sn);
  }
  __syncthreads();

  const cx<T>* px = ptab;
  const cx<T>* py = ptab + w0;
  const cx<T>* pz = ptab + w0 + w1;
  const P4* __restrict__ C2 = reinterpret_cast<const P4*>(a.C2p);
  const cx<T>* __restrict__ C1 = reinterpret_cast<const cx<T>*>(a.C1);
  const int sy = w2 + 1, sx = (w1 + 2) * (w2 + 1);
  const T eps = (T)a.tie_eps;
  const int p = sp.p, q = sp.q, r = sp.r;
  const int wp = p == 0 ? w0 : (p == 1 ? w1 : w2);
  const int wq = q == 0 ? w0 : (q == 1 ? w1 : w2);
  const int wr = r == 0 ? w0 : (r == 1 ? w1 : w2);
  const T m00 = (T)sp.mu[0][0], m01 = (T)sp.mu[0][1], m02 = (T)sp.mu[0][2];
  const T m10 = (T)sp.mu[1][0], m11 = (T)sp.mu[1][1], m12 = (T)sp.mu[1][2];
  const T m20 = (T)sp.mu[2][0], m21 = (T)sp.mu[2][1], m22 = (T)sp.mu[2][2];
  const int lane = tid & 31, warp = tid >> 5;
  const int dp = 4 * (warp & 3) + (lane & 3);
  const int dq = 8 * (warp >> 2) + (lane >> 2);
  const int units = sp.nP * sp.nQ * wr;

  Acc26<T> acc;
  acc.zero();
  for (int unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int kr = unit % wr;
    const int iq = (unit / wr) % sp.nQ;
    const int ip = unit / (wr * sp.nQ);
    const int kp = 16 * ip + dp, kq = 16 * iq + dq;
    if (kp >= wp || kq >= wq) continue;
    const int kx = p == 0 ? kp : (q == 0 ? kq : kr);
    const int ky = p == 1 ? kp : (q == 1 ? kq : kr);
    const int kz = p == 2 ? kp : (q == 2 ? kq : kr);
    const T kapx = (T)(kx - hx), kapy = (T)(ky - hy), kapz = (T)(kz - hz);
    T u[3] = {fma(m02, kapz, fma(m01, kapy, fma(m00, kapx, (T)hx))),
              fma(m12, kapz, fma(m11, kapy, fma(m10, kapx, (T)hy))),
              fma(m22, kapz, fma(m21, kapy, fma(m20, kapx, (T)hz)))};
    T fl[3], f[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      fl[ax] = floor(u[ax]);
      f[ax] = u[ax] - fl[ax];
    }
    const bool tz = a.dim == 3 && (f[2] < eps || f[2] > (T)1 - eps);
    if (f[0] < eps || f[0] > (T)1 - eps || f[1] < eps || f[1] > (T)1 - eps || tz) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        if ((ax < 2 || tz) && (f[ax] < eps || f[ax] > (T)1 - eps)) {
          double ue = exact_u_s(sp.R, a.dom, ax, kx, ky, kz, hx, hy, hz, ax == 0 ? hx : (ax == 1 ? hy : hz));
          double fe = floor(ue);
          fl[ax] = (T)fe;
          f[ax] = (T)(ue - fe);
        }
      }
    }
    int ix = (int)fl[0], iy = (int)fl[1], iz = (int)fl[2];
    if (WRAP) {
      ix = ix < 0 ? ix + w0 : (ix >= w0 ? ix - w0 : ix);
      iy = iy < 0 ? iy + w1 : (iy >= w1 ? iy - w1 : iy);
      iz = iz < 0 ? iz + w2 : (iz >= w2 ? iz - w2 : iz);
    } else if ((unsigned)(ix + 1) > (unsigned)w0 || (unsigned)(iy + 1) > (unsigned)w1 ||
               (unsigned)(iz + 1) > (unsigned)w2) {
      continue;
    }
    const P4* ptr = C2 + ((ix + 1) * sx + (iy + 1) * sy + (iz + 1));
    P4 e00 = ldg_pair(ptr), e10 = ldg_pair(ptr + sx), e01 = ldg_pair(ptr + sy), e11 = ldg_pair(ptr + sx + sy);
    const cx<T> base = C1[(kx * w1 + ky) * w2 + kz] * ((px[kx] * py[ky]) * pz[kz]);
    const T fu = f[0], fv = f[1], fs = f[2];
    cx<T> c000 = mk<T>(e00.x, e00.y), c001 = mk<T>(e00.z, e00.w);
    cx<T> c100 = mk<T>(e10.x, e10.y), c101 = mk<T>(e10.z, e10.w);
    cx<T> c010 = mk<T>(e01.x, e01.y), c011 = mk<T>(e01.z, e01.w);
    cx<T> c110 = mk<T>(e11.x, e11.y), c111 = mk<T>(e11.z, e11.w);
    cx<T> d00 = c100 - c000, d01 = c101 - c001, d10 = c110 - c010, d11 = c111 - c011;
    cx<T> a00 = mk<T>(fma(fu, d00.re, c000.re), fma(fu, d00.im, c000.im));
    cx<T> a01 = mk<T>(fma(fu, d01.re, c001.re), fma(fu, d01.im, c001.im));
    cx<T> a10 = mk<T>(fma(fu, d10.re, c010.re), fma(fu, d10.im, c010.im));
    cx<T> a11 = mk<T>(fma(fu, d11.re, c011.re), fma(fu, d11.im, c011.im));
    cx<T> b0 = lerp(a00, a10, fv), b1 = lerp(a01, a11, fv);
    cx<T> V = lerp(b0, b1, fs);
    cx<T> dU = lerp(lerp(d00, d10, fv), lerp(d01, d11, fv), fs);
    cx<T> dV = lerp(a10 - a00, a11 - a01, fs);
    cx<T> dS = b1 - b0;
    cx<T> bV = base * V;
    acc.add(bV, base * dU, base * dV, base * dS, kapx, kapy, kapz);
  }

  // ---- block reduction through a shared-memory transpose (fixed order)
#pragma unroll
  for (int c = 0; c < kNumMoments; ++c) tr[c][tid] = acc.v[c];
  __syncthreads();
  // 26 moments x 8 segments of 32 values: thread (c, s) sums its segment
  double part = 0.0;
  const int c = tid >> 3, s = tid & 7;
  if (c < kNumMoments) {
    T acc2 = (T)0;
#pragma unroll 8
    for (int i = 0; i < 32; ++i) acc2 += tr[c][s * 32 + i];
    part = (double)acc2;
  }
  // combine the 8 segments of each moment (lanes 8 apart inside one warp)
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o, 8);
  if (c < kNumMoments && s == 0) red[c] = part;
  __syncthreads();

  double* out = a.out;
  const int bpp = gridDim.x;
  if (bpp == 1) {
    if (tid < 14) out[tid] = finalize_slot(a, sp.R, red, tid);
    return;
  }
  double* pt = a.partials + (int64_t)blockIdx.x * kNumMoments;
  if (tid < kNumMoments) pt[tid] = red[tid];
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(a.counters, 1u);
  __syncthreads();
  if (ticket != (unsigned)(bpp - 1)) return;
  __threadfence();
  // last block: 26 moments x 9 segments; each thread streams its segment's
  // partials with independent loads (fixed order), then segments combine
  if (tid < kNumMoments * 9) {
    const int cc = tid / 9, sg = tid % 9;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    int b = sg;
    for (; b + 27 < bpp; b += 36) {
      v0 += __ldcg(a.partials + (int64_t)b * kNumMoments + cc);
      v1 += __ldcg(a.partials + (int64_t)(b + 9) * kNumMoments + cc);
      v2 += __ldcg(a.partials + (int64_t)(b + 18) * kNumMoments + cc);
      v3 += __ldcg(a.partials + (int64_t)(b + 27) * kNumMoments + cc);
    }
    for (; b < bpp; b += 9) v0 += __ldcg(a.partials + (int64_t)b * kNumMoments + cc);
    reinterpret_cast<double*>(&tr[0][0])[tid] = (v0 + v1) + (v2 + v3);
  }
  __syncthreads();
  if (tid < kNumMoments) {
    const double* seg = reinterpret_cast<const double*>(&tr[0][0]) + tid * 9;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) v += seg[k];
    red[tid] = v;
  }
  __syncthreads();
  if (tid < 14) out[tid] = finalize_slot(a, sp.R, red, tid);
  if (tid == 0) a.counters[0] = 0u;
}

template <typename T, bool WRAP>
cudaError_t launch_single_t(const CascadeArgs& a, cudaStream_t st) {
  size_t smem = sizeof(T) * kNumMoments * (kThreads + 1) + 16 + sizeof(cx<T>) * (a.w[0] + a.w[1] + a.w[2]);
  static size_t configured = 0;
  if (smem > configured && smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(cascade3d_single_kernel<T, WRAP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  cascade3d_single_kernel<T, WRAP><<<a.blocks_per_pose, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

int single_blocks(const CascadeArgs& a, int sms) {
  // units = nP * nQ * w_r, bounded by the orientation-independent worst case
  int64_t best = 0;
  for (int r = 0; r < 3; ++r) {
    int o1 = (r + 1) % 3, o2 = (r + 2) % 3;
    int64_t u = ceil_div(a.w[o1], 16) * ceil_div(a.w[o2], 16) * a.w[r];
    if (best == 0 || u < best) best = u;
  }
  int64_t target = (int64_t)sms * (a.precision == 32 ? 3 : 2);
  if (const char* env = getenv("GF_SINGLE_BLOCKS")) target = atoi(env);  // experiments only
  return (int)(best < target ? best : target);
}

cudaError_t launch_cascade_single(const CascadeArgs& a, cudaStream_t st) {
  if (a.precision == 32) return a.wrap ? launch_single_t<float, true>(a, st) : launch_single_t<float, false>(a, st);
  return a.wrap ? launch_single_t<double, true>(a, st) : launch_single_t<double, false>(a, st);
}

}  // namespace gf
