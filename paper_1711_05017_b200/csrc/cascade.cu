// cascade.cu -- the per-pose energy/force/torque query (Q1) and the batched
// pose sweep (Q3) on sm_100a.
//
// Semantics follow the reference kernel _core.cascade_3d
// (/root/reference/pkg/src/geofield/_core.pyx:598-724): for every retained
// window mode k the moving window C2 is trilinearly sampled at the rotated
// continuous index u = -R^T w / dw + w/2 (zero outside the window unless
// `wrap`, periodic otherwise), multiplied by C1(k) and the translation phase
// exp(2 pi i w.t_eff), and seven complex sums are formed: the score, the
// three translational derivatives and the three rotational derivatives
// (analytic trilinear gradient, generators Omega_x,y,z).
//
// B200 design:
//  * C2 is stored zero- (or periodically-) padded by one cell and packed so
//    that one 16-byte (fp32) / 32-byte (fp64) load returns the z-pair
//    (c[i][j][k], c[i][j][k+1]); a mode's 8-corner footprint is 4 loads with
//    no bounds tests.  Modes whose footprint lies wholly outside a truncated
//    window contribute exact zeros and are skipped (bit-safe).
//  * Each thread owns a run of L consecutive kz modes: the continuous index
//    is one FMA per axis per mode, and the translation phase advances by a
//    sincospi-seeded complex recurrence (one sincospi per run, not per mode).
//  * Instead of the reference's seven per-mode complex products, each mode
//    adds base*V and base*dV/du_b into 26 moment accumulators
//    (sum bV, sum bV k_a, sum b dV_b k_a); the seven outputs are exact linear
//    combinations of these moments, formed once per pose in float64.
//  * Floor decisions reproduce the reference bit for bit: where the fast
//    index lies within a few ulps of an integer the index is recomputed with
//    the reference's float64 operation order (no FMA contraction), so the
//    trilinear cell -- and hence the torque slope -- matches even at lattice
//    rotations.
//  * Reductions are fixed-order trees (warp shuffles, then float64 across
//    warps and blocks, last-block-done with an integer ticket): repeated calls
//    are bitwise identical; no float atomics anywhere.
#include "common.cuh"
#include "cascade.cuh"

#include <math.h>

namespace gf {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct PoseShared {
  double mu[3][3];   // u_a = h_a + sum_b mu[a][b] * kappa_b
  double targ[3];    // cycles of exp(2 pi i w.t) per unit kappa_a: dw_a * t_a
  double R[9];
  double step_re, step_im;  // exp(2 pi i targ[2])
};

__device__ __forceinline__ void load_pose(const CascadeArgs& a, int64_t p, PoseShared& ps) {
  // one warp fills the per-pose constants
  const double* src = a.poses ? a.poses + p * 12 : a.pose_inline;
  int t = threadIdx.x;
  if (t < 9) ps.R[t] = src[t];
  __syncwarp();
  if (t < 9) {
    int ia = t / 3, ib = t % 3;
    // nu_a = -sum_b R[b][a] w_b ; u_a = nu_a / dw_a + h_a, w_b = kappa_b dw_b
    ps.mu[ia][ib] = -src[ib * 3 + ia] * (a.dom[ib] / a.dom[ia]);
  }
  if (t >= 16 && t < 19) ps.targ[t - 16] = a.dom[t - 16] * src[9 + t - 16];
  if (t == 20) {
    double s, c;
    sincospi(2.0 * (a.dom[2] * src[11] - rint(a.dom[2] * src[11])), &s, &c);
    ps.step_re = c;
    ps.step_im = s;
  }
}

// Reference-order float64 continuous index for one axis (_core.pyx:633-643):
// om_b = (k_b - h_b) * dw_b ; nu = -(R[0][a] om_x + R[1][a] om_y + R[2][a] om_z)
// u = nu / dw_a + h_a, every operation separately rounded.
__device__ __forceinline__ double exact_u(const PoseShared& ps, const double* dom, int a, int kx, int ky,
                                          int kz, int hx, int hy, int hz, int ha) {
  double ox = __dmul_rn((double)(kx - hx), dom[0]);
  double oy = __dmul_rn((double)(ky - hy), dom[1]);
  double oz = __dmul_rn((double)(kz - hz), dom[2]);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(ps.R[0 + a], ox), __dmul_rn(ps.R[3 + a], oy)),
                       __dmul_rn(ps.R[6 + a], oz));
  return __dadd_rn(__ddiv_rn(-s, dom[a]), (double)ha);
}

template <typename T> struct Acc {
  cx<T> S;       // sum bV
  cx<T> Z[3];    // sum bV kappa_a
  cx<T> Y[3][3]; // sum b dV_b kappa_a   (index [b][a])
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Reduce the 26 moments across the block in a fixed order; result (float64)
// lands in red[0..25] (shared) for thread 0's block.
template <typename T>
__device__ __forceinline__ void block_reduce(const Acc<T>& acc, double (*wsum)[kNumMoments], double* red) {
  const T* v = reinterpret_cast<const T*>(&acc);
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < kNumMoments; ++c) {
    T s = warp_sum(v[c]);
    if (lane == 0) wsum[warp][c] = (double)s;
  }
  __syncthreads();
  if (threadIdx.x < kNumMoments) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += wsum[w][threadIdx.x];
    red[threadIdx.x] = s;
  }
  __syncthreads();
}

// Form the seven outputs from the moments (float64), times dcell.
__device__ void finalize(const CascadeArgs& a, const PoseShared& ps, const double* m, double* out) {
  const double TWO_PI = 6.283185307179586;
  if (threadIdx.x != 0) return;
  const double* R = ps.R;
  double dc = a.dcell;
  out[0] = dc * m[0];
  out[1] = dc * m[1];
  for (int ax = 0; ax < 3; ++ax) {  // T_a = 2 pi i dw_a Z_a
    double zr = m[2 + 2 * ax], zi = m[3 + 2 * ax], k = dc * TWO_PI * a.dom[ax];
    out[2 + 2 * ax] = -k * zi;
    out[3 + 2 * ax] = k * zr;
  }
  // A_g = Omega_g R (_core.pyx:615-626), q_g = A_g c
  double A[3][3][3] = {};
  for (int b = 0; b < 3; ++b) {
    A[0][1][b] = -R[6 + b]; A[0][2][b] = R[3 + b];
    A[1][0][b] = R[6 + b];  A[1][2][b] = -R[0 + b];
    A[2][0][b] = -R[3 + b]; A[2][1][b] = R[0 + b];
  }
  for (int g = 0; g < 3; ++g) {
    double gr = 0.0, gi = 0.0;
    // - sum_{b,a} A_g[a][b] (dw_a / dw_b) Y[b][a]
    for (int b = 0; b < 3; ++b)
      for (int ax = 0; ax < 3; ++ax) {
        double coef = -A[g][ax][b] * (a.dom[ax] / a.dom[b]);
        gr += coef * m[8 + 2 * (3 * b + ax)];
        gi += coef * m[9 + 2 * (3 * b + ax)];
      }
    // + 2 pi i sum_a dw_a q_g[a] Z_a
    for (int ax = 0; ax < 3; ++ax) {
      double q = A[g][ax][0] * a.center[0] + A[g][ax][1] * a.center[1] + A[g][ax][2] * a.center[2];
      double k = TWO_PI * a.dom[ax] * q;
      gr += -k * m[3 + 2 * ax];
      gi += k * m[2 + 2 * ax];
    }
    out[8 + 2 * g] = dc * gr;
    out[9 + 2 * g] = dc * gi;
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) cascade3d_kernel(CascadeArgs a) {
  using P4 = typename pair4<T>::type;
  __shared__ PoseShared ps;
  __shared__ double wsum[kWarps][kNumMoments];
  __shared__ double red[kNumMoments];
  __shared__ unsigned ticket;

  const int bpp = a.blocks_per_pose;
  const int64_t pose = a.pose_offset + blockIdx.x / bpp;
  const int blk = blockIdx.x % bpp;

  if (threadIdx.x < 32) load_pose(a, pose, ps);
  __syncthreads();

  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  const int L = a.seg_len;
  const int spr = a.segs_per_row;
  const int64_t sy = (int64_t)(w2 + 1), sx = (int64_t)(w1 + 2) * (w2 + 1);
  const P4* __restrict__ C2 = reinterpret_cast<const P4*>(a.C2p);
  const cx<T>* __restrict__ C1 = reinterpret_cast<const cx<T>*>(a.C1);
  const T eps = (T)a.tie_eps;
  const T mz0 = (T)ps.mu[0][2], mz1 = (T)ps.mu[1][2], mz2 = (T)ps.mu[2][2];
  const cx<T> step = mk<T>((T)ps.step_re, (T)ps.step_im);

  Acc<T> acc;
  {
    T* v = reinterpret_cast<T*>(&acc);
#pragma unroll
    for (int c = 0; c < kNumMoments; ++c) v[c] = (T)0;
  }

  const int64_t seg_begin = (int64_t)blk * a.segs_per_block;
  int64_t seg_end = seg_begin + a.segs_per_block;
  if (seg_end > a.n_seg) seg_end = a.n_seg;

  for (int64_t s = seg_begin + threadIdx.x; s < seg_end; s += kThreads) {
    const int row = (int)(s / spr);
    const int kz0 = (int)(s - (int64_t)row * spr) * L;
    const int kx = row / w1, ky = row - (row / w1) * w1;
    const int kend = min(kz0 + L, w2);
    const double kapx = kx - hx, kapy = ky - hy, kapz0 = kz0 - hz;
    // run start: continuous indices (float64 -> T) and phase seed
    const T u0x = (T)(hx + ps.mu[0][0] * kapx + ps.mu[0][1] * kapy + ps.mu[0][2] * kapz0);
    const T u0y = (T)(hy + ps.mu[1][0] * kapx + ps.mu[1][1] * kapy + ps.mu[1][2] * kapz0);
    const T u0z = (T)(hz + ps.mu[2][0] * kapx + ps.mu[2][1] * kapy + ps.mu[2][2] * kapz0);
    cx<T> ph;
    {
      double cyc = ps.targ[0] * kapx + ps.targ[1] * kapy + ps.targ[2] * kapz0;
      cyc -= rint(cyc);
      T sn, cs;
      if constexpr (sizeof(T) == 4) sincospif(2.0f * (float)cyc, &sn, &cs);
      else sincospi(2.0 * cyc, &sn, &cs);
      ph = mk<T>(cs, sn);
    }
    // per-run partial moments (kappa_x, kappa_y are constant along the run)
    cx<T> rS = mk<T>(0, 0), rZz = mk<T>(0, 0);
    cx<T> rX[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
    cx<T> rXz[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
    const cx<T>* c1row = C1 + ((int64_t)kx * w1 + ky) * w2;

    for (int kz = kz0; kz < kend; ++kz) {
      const T j = (T)(kz - kz0);
      T u[3] = {fma(j, mz0, u0x), fma(j, mz1, u0y), fma(j, mz2, u0z)};
      T fl[3], f[3];
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        fl[ax] = floor(u[ax]);
        f[ax] = u[ax] - fl[ax];
      }
      // near an integer: take the reference's float64 floor decision
      const bool tz = a.dim == 3 && (f[2] < eps || f[2] > (T)1 - eps);
      if (f[0] < eps || f[0] > (T)1 - eps || f[1] < eps || f[1] > (T)1 - eps || tz) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          if ((ax < 2 || tz) && (f[ax] < eps || f[ax] > (T)1 - eps)) {
            double ue = exact_u(ps, a.dom, ax, kx, ky, kz, hx, hy, hz, ax == 0 ? hx : (ax == 1 ? hy : hz));
            double fe = floor(ue);
            fl[ax] = (T)fe;
            f[ax] = (T)(ue - fe);
          }
        }
      }
      const cx<T> phk = ph;
      ph = ph * step;
      int ix = (int)fl[0], iy = (int)fl[1], iz = (int)fl[2];
      if (a.wrap) {
        ix = ix < 0 ? ix + w0 : (ix >= w0 ? ix - w0 : ix);
        iy = iy < 0 ? iy + w1 : (iy >= w1 ? iy - w1 : iy);
        iz = iz < 0 ? iz + w2 : (iz >= w2 ? iz - w2 : iz);
      } else if (ix < -1 || ix > w0 - 1 || iy < -1 || iy > w1 - 1 || iz < -1 || iz > w2 - 1) {
        continue;  // whole footprint outside the window: exact zero contribution
      }
      const cx<T> base = c1row[kz] * phk;
      const P4* p = C2 + (int64_t)(ix + 1) * sx + (int64_t)(iy + 1) * sy + (iz + 1);
      P4 e00 = ldg_pair(p), e10 = ldg_pair(p + sx), e01 = ldg_pair(p + sy), e11 = ldg_pair(p + sx + sy);
      // corners c[x][y][z]: e{x}{y} = (c[x][y][0], c[x][y][1])
      const T fu = f[0], fv = f[1], fs = f[2];
      cx<T> c000 = mk<T>(e00.x, e00.y), c001 = mk<T>(e00.z, e00.w);
      cx<T> c100 = mk<T>(e10.x, e10.y), c101 = mk<T>(e10.z, e10.w);
      cx<T> c010 = mk<T>(e01.x, e01.y), c011 = mk<T>(e01.z, e01.w);
      cx<T> c110 = mk<T>(e11.x, e11.y), c111 = mk<T>(e11.z, e11.w);
      // along x: a_yz, d_yz = c1yz - c0yz
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
      cx<T> X0 = base * dU, X1 = base * dV, X2 = base * dS;
      const T kz_k = (T)(kz - hz);
      rS += bV;
      axpy(rZz, kz_k, bV);
      rX[0] += X0; rX[1] += X1; rX[2] += X2;
      axpy(rXz[0], kz_k, X0); axpy(rXz[1], kz_k, X1); axpy(rXz[2], kz_k, X2);
    }
    const T kxk = (T)kapx, kyk = (T)kapy;
    acc.S += rS;
    axpy(acc.Z[0], kxk, rS);
    axpy(acc.Z[1], kyk, rS);
    acc.Z[2] += rZz;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      axpy(acc.Y[b][0], kxk, rX[b]);
      axpy(acc.Y[b][1], kyk, rX[b]);
      acc.Y[b][2] += rXz[b];
    }
  }

  block_reduce<T>(acc, wsum, red);

  double* out = a.out + pose * 14;
  if (bpp == 1) {
    finalize(a, ps, red, out);
    return;
  }
  // cross-block: publish this block's moments, last block reduces in fixed order
  double* part = a.partials + (pose * bpp + blk) * kNumMoments;
  if (threadIdx.x < kNumMoments) part[threadIdx.x] = red[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(a.counters + pose, 1u);
  __syncthreads();
  if (ticket != (unsigned)(bpp - 1)) return;
  __threadfence();
  const double* base = a.partials + pose * bpp * kNumMoments;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < kNumMoments; c += kWarps) {
    double s = 0.0;
    for (int b = lane; b < bpp; b += 32) s += __ldcg(base + (int64_t)b * kNumMoments + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[c] = s;
  }
  __syncthreads();
  finalize(a, ps, red, out);
  if (threadIdx.x == 0) a.counters[pose] = 0u;  // re-arm for the next launch
}

// Build the padded + z-pair-packed copy of a window for use as the moving
// operand.  Source: raw complex<T> window (w0, w1, w2).  Destination:
// (w0+2) x (w1+2) x (w2+1) pairs; padded index P = window index + 1; the
// border is zero (truncated windows) or the periodic image (full spectra).
template <typename T>
__global__ void pack_window_kernel(const cx<T>* __restrict__ src, typename pair4<T>::type* __restrict__ dst,
                                   int w0, int w1, int w2, int wrap) {
  int64_t n = (int64_t)(w0 + 2) * (w1 + 2) * (w2 + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    int K = (int)(e % (w2 + 1));
    int64_t r = e / (w2 + 1);
    int J = (int)(r % (w1 + 2));
    int I = (int)(r / (w1 + 2));
    auto fetch = [&](int i, int j, int k) -> cx<T> {
      if (wrap) {
        i = (i + w0) % w0; j = (j + w1) % w1; k = (k + w2) % w2;
      } else if (i < 0 || i >= w0 || j < 0 || j >= w1 || k < 0 || k >= w2) {
        return mk<T>(0, 0);
      }
      return src[((int64_t)i * w1 + j) * w2 + k];
    };
    cx<T> lo = fetch(I - 1, J - 1, K - 1), hi = fetch(I - 1, J - 1, K);
    typename pair4<T>::type v;
    v.x = lo.re; v.y = lo.im; v.z = hi.re; v.w = hi.im;
    dst[e] = v;
  }
}

template <typename T>
__global__ void narrow_kernel(const cx<double>* __restrict__ src, cx<T>* __restrict__ dst, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = mk<T>((T)src[e].re, (T)src[e].im);
}

}  // namespace

int64_t packed_window_elems(const int w[3]) { return (int64_t)(w[0] + 2) * (w[1] + 2) * (w[2] + 1); }

cudaError_t launch_pack_window(int precision, const void* raw, void* packed, const int w[3], int wrap,
                               cudaStream_t st) {
  int64_t n = packed_window_elems(w);
  int grid = (int)ceil_div(n, 256);
  if (grid > 148 * 16) grid = 148 * 16;
  if (precision == 32)
    pack_window_kernel<float><<<grid, 256, 0, st>>>((const cx<float>*)raw, (float4*)packed, w[0], w[1], w[2], wrap);
  else
    pack_window_kernel<double><<<grid, 256, 0, st>>>((const cx<double>*)raw, (double4*)packed, w[0], w[1], w[2], wrap);
  return cudaGetLastError();
}

cudaError_t launch_narrow(const void* src, void* dst, int64_t n, cudaStream_t st) {
  int grid = (int)ceil_div(n, 256);
  if (grid > 148 * 16) grid = 148 * 16;
  narrow_kernel<float><<<grid, 256, 0, st>>>((const cx<double>*)src, (cx<float>*)dst, n);
  return cudaGetLastError();
}

void plan_cascade(CascadeArgs& a, int64_t n_poses, int target_blocks) {
  // run length: L modes along kz per thread (divides work evenly when possible)
  int w2 = a.w[2];
  int L = a.seg_len > 0 ? a.seg_len : 8;
  if (L > w2) L = w2;
  a.seg_len = L;
  a.segs_per_row = (int)ceil_div(w2, L);
  a.n_seg = (int64_t)a.w[0] * a.w[1] * a.segs_per_row;
  int64_t max_bpp = ceil_div(a.n_seg, kThreads);
  int64_t bpp = 1;
  if (n_poses < target_blocks) bpp = ceil_div(target_blocks, n_poses);
  if (bpp > max_bpp) bpp = max_bpp;
  if (bpp < 1) bpp = 1;
  a.blocks_per_pose = (int)bpp;
  a.segs_per_block = ceil_div(a.n_seg, bpp);
  // tie zone: several ulps of the largest |u| reachable at this geometry
  double umax = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    double s = a.w[ax] / 2;
    for (int b = 0; b < 3; ++b) s += (a.dom[b] / a.dom[ax]) * (a.w[b] / 2 + 1);
    if (s > umax) umax = s;
  }
  double ulp = (a.precision == 32) ? ldexp(umax, -23) : ldexp(umax, -52);
  double eps = 8.0 * ulp;
  double floor_eps = (a.precision == 32) ? 1e-4 : 1e-9;
  a.tie_eps = eps > floor_eps ? eps : floor_eps;
}

cudaError_t launch_cascade(const CascadeArgs& a, int64_t n_poses, cudaStream_t st) {
  // grid.x = poses x blocks_per_pose, issued in chunks that fit gridDim.x
  const int64_t max_blocks = (int64_t)1 << 30;
  int64_t chunk = max_blocks / a.blocks_per_pose;
  for (int64_t p0 = 0; p0 < n_poses; p0 += chunk) {
    int64_t np = n_poses - p0 < chunk ? n_poses - p0 : chunk;
    CascadeArgs c = a;
    c.pose_offset = a.pose_offset + p0;
    unsigned grid = (unsigned)(np * a.blocks_per_pose);
    if (a.precision == 32)
      cascade3d_kernel<float><<<grid, kThreads, 0, st>>>(c);
    else
      cascade3d_kernel<double><<<grid, kThreads, 0, st>>>(c);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace gf
