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
#include <stdlib.h>

#include <type_traits>

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

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
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

// Direct-gather kernel.  Lane layout: each warp owns a 4 x 8 patch of modes
// in the (p, q) mode plane and every lane walks a run of L modes along the
// third axis r.  Per pose, r is the mode axis whose rotated image has the
// smallest C2-z component, i.e. the patch plane is the one whose image lies
// closest to C2's z lines: the 32 lanes' corner pairs then share far fewer
// 128-byte lines per load (one L1 wavefront per distinct line).
struct Orient {
  int p, q, r;        // mode axes: 4-lane, 8-lane, run
  int nP, nQ, nR;     // patch tiles (16 wide) along p, q and runs along r
  double step_re[3], step_im[3];
};

// fp32: four resident CTAs per SM (64 registers; the spilled values are
// per-pose constants, L1-resident): the L2-resident gathers are latency
// bound, and twice the warps gain 14-15 % poses/s at w = 64-128 over two CTAs
// (five or more collapse under spills; profiles/r02_sweep_orientation.txt)
template <typename T, bool WRAP>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? 4 : 2) cascade3d_kernel(CascadeArgs a) {
  using P4 = typename pair4<T>::type;
  __shared__ PoseShared ps;
  __shared__ Orient orient;
  __shared__ double wsum[kWarps][kNumMoments];
  __shared__ double red[kNumMoments];
  __shared__ unsigned ticket;
  __shared__ int tie_dep[3];
  // tie table (lattice-aligned poses, see cascade_single.cu): (floor, frac)
  // of the reference index of axis c at [offset(b) + k_b] when column c of R
  // has its single nonzero in row b
  extern __shared__ __align__(16) unsigned char dyn_smem[];
  cx<T>* ttab = reinterpret_cast<cx<T>*>(dyn_smem);

  const int bpp = a.blocks_per_pose;
  const int64_t pose = a.pose_offset + blockIdx.x / bpp;
  const int blk = blockIdx.x % bpp;
  const int tid = threadIdx.x;
  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int L = a.seg_len;

  if (tid < 32) load_pose(a, pose, ps);
  __syncthreads();
  if (tid == 0) {
    // run axis r: smallest |R[b][2]| (equal spacing: C2-z component of mode
    // axis b), but never z: a run along C1's contiguous axis puts the 32 lanes
    // of every C1 load on 32 different lines (measured +3.5-4 % over all
    // cmd_bench poses at w = 64/96/128 against the unrestricted choice, and
    // ahead of a per-pose line-count model, profiles/r02_sweep_orientation.txt)
    int r = 2;
    if (a.dim == 3) {
      double z[3] = {fabs(ps.mu[2][0]), fabs(ps.mu[2][1]), fabs(ps.mu[2][2])};
      r = z[0] <= z[1] ? 0 : 1;
    }
    int o1 = (r + 1) % 3, o2 = (r + 2) % 3;
    if (a.dim == 2) { o1 = 0; o2 = 1; }
    // the 8-lane axis q is the one whose image is most aligned with C2-z
    bool swap = fabs(ps.mu[2][o1]) > fabs(ps.mu[2][o2]);
    orient.p = swap ? o2 : o1;
    orient.q = swap ? o1 : o2;
    orient.r = r;
    const int wv[3] = {w0, w1, w2};
    orient.nP = (wv[orient.p] + 15) / 16;
    orient.nQ = (wv[orient.q] + 15) / 16;
    orient.nR = (wv[r] + L - 1) / L;
    for (int ax = 0; ax < 3; ++ax) {
      double s, c;
      double t = ps.targ[ax];
      sincospi(2.0 * (t - rint(t)), &s, &c);
      orient.step_re[ax] = c;
      orient.step_im[ax] = s;
    }
  }
  if (tid == 32) {
    for (int ax = 0; ax < 3; ++ax) {
      const double* R = ps.R;
      const int nz = (R[ax] != 0.0) + (R[3 + ax] != 0.0) + (R[6 + ax] != 0.0);
      tie_dep[ax] = nz != 1 ? -1 : (R[ax] != 0.0 ? 0 : (R[3 + ax] != 0.0 ? 1 : 2));
    }
  }
  __syncthreads();
  if (tie_dep[0] >= 0 || tie_dep[1] >= 0 || tie_dep[2] >= 0) {
    for (int i = tid; i < w0 + w1 + w2; i += kThreads) {
      const int b = i < w0 ? 0 : (i < w0 + w1 ? 1 : 2);
      const int k = i - (b == 0 ? 0 : (b == 1 ? w0 : w0 + w1));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        if (tie_dep[c] != b) continue;
        const double ue = exact_u(ps, a.dom, c, b == 0 ? k : w0 / 2, b == 1 ? k : w1 / 2, b == 2 ? k : w2 / 2, w0 / 2,
                                  w1 / 2, w2 / 2, c == 0 ? w0 / 2 : (c == 1 ? w1 / 2 : w2 / 2));
        const double fe = floor(ue);
        ttab[i] = mk<T>((T)fe, (T)(ue - fe));
      }
    }
    __syncthreads();
  }

  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  const int64_t sy = (int64_t)(w2 + 1), sx = (int64_t)(w1 + 2) * (w2 + 1);
  const P4* __restrict__ C2 = reinterpret_cast<const P4*>(a.C2p);
  const cx<T>* __restrict__ C1 = reinterpret_cast<const cx<T>*>(a.C1);
  const T eps = (T)a.tie_eps;
  const int p = orient.p, q = orient.q, r = orient.r;
  const int wp = p == 0 ? w0 : (p == 1 ? w1 : w2);
  const int wq = q == 0 ? w0 : (q == 1 ? w1 : w2);
  const int wr = r == 0 ? w0 : (r == 1 ? w1 : w2);
  const int sr = r == 0 ? w1 * w2 : (r == 1 ? w2 : 1);
  const T mr0 = (T)ps.mu[0][r], mr1 = (T)ps.mu[1][r], mr2 = (T)ps.mu[2][r];
  const cx<T> step = mk<T>((T)orient.step_re[r], (T)orient.step_im[r]);
  const T er0 = r == 0 ? (T)1 : (T)0, er1 = r == 1 ? (T)1 : (T)0, er2 = r == 2 ? (T)1 : (T)0;
  const int lane = tid & 31, warp = tid >> 5;
  const int dp = 4 * (warp & 3) + (lane & 3);
  const int dq = 8 * (warp >> 2) + (lane >> 2);
  const int units = orient.nP * orient.nQ * orient.nR;

  const int tmask = (tie_dep[0] >= 0 ? 1 : 0) | (tie_dep[1] >= 0 ? 2 : 0) | (a.dim == 3 && tie_dep[2] >= 0 ? 4 : 0);
  Acc26<T> acc;
  acc.zero();

  // the unit loop, compiled twice: with the tie table (lattice-aligned pose)
  // and without it (generic pose: no table branch in the mode loop)
  auto unit_loop = [&](auto ties_c) {
  constexpr bool TIES = decltype(ties_c)::value;
  for (int unit = blk; unit < units; unit += bpp) {
    const int ir = unit % orient.nR;
    const int iq = (unit / orient.nR) % orient.nQ;
    const int ip = unit / (orient.nR * orient.nQ);
    const int kp = 16 * ip + dp, kq = 16 * iq + dq, kr0 = L * ir;
    if (kp >= wp || kq >= wq) continue;
    const int kend = min(kr0 + L, wr);
    const int kx = p == 0 ? kp : (q == 0 ? kq : kr0);
    const int ky = p == 1 ? kp : (q == 1 ? kq : kr0);
    const int kz0 = p == 2 ? kp : (q == 2 ? kq : kr0);
    const double kap[3] = {(double)(kx - hx), (double)(ky - hy), (double)(kz0 - hz)};
    const T u0x = (T)(hx + ps.mu[0][0] * kap[0] + ps.mu[0][1] * kap[1] + ps.mu[0][2] * kap[2]);
    const T u0y = (T)(hy + ps.mu[1][0] * kap[0] + ps.mu[1][1] * kap[1] + ps.mu[1][2] * kap[2]);
    const T u0z = (T)(hz + ps.mu[2][0] * kap[0] + ps.mu[2][1] * kap[1] + ps.mu[2][2] * kap[2]);
    cx<T> ph;
    {
      double cyc = ps.targ[0] * kap[0] + ps.targ[1] * kap[1] + ps.targ[2] * kap[2];
      cyc -= rint(cyc);
      T sn, cs;
      if constexpr (sizeof(T) == 4) sincospif(2.0f * (float)cyc, &sn, &cs);
      else sincospi(2.0 * cyc, &sn, &cs);
      ph = mk<T>(cs, sn);
    }
    cx<T> rS = mk<T>(0, 0), rJ = mk<T>(0, 0);
    cx<T> rX[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
    cx<T> rXJ[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
    int c1off = (kx * w1 + ky) * w2 + kz0;

    for (int kr = kr0; kr < kend; ++kr, c1off += sr) {
      const T j = (T)(kr - kr0);
      T u[3] = {fma(j, mr0, u0x), fma(j, mr1, u0y), fma(j, mr2, u0z)};
      T fl[3], f[3];
      bool tie[3];
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        fl[ax] = floor(u[ax]);
        f[ax] = u[ax] - fl[ax];
        tie[ax] = !(TIES && ((tmask >> ax) & 1)) && (ax < 2 || a.dim == 3) && (f[ax] < eps || f[ax] > (T)1 - eps);
      }
      if (TIES || tie[0] || tie[1] || tie[2]) {
        const int kkx = r == 0 ? kr : kx, kky = r == 1 ? kr : ky, kkz = r == 2 ? kr : kz0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          if (TIES && ((tmask >> ax) & 1)) {  // lattice-aligned axis: tabulated reference floor / frac
            const int dep = tie_dep[ax];
            const cx<T> e = ttab[dep == 0 ? kkx : (dep == 1 ? w0 + kky : w0 + w1 + kkz)];
            fl[ax] = e.re;
            f[ax] = e.im;
          } else if (tie[ax]) {  // reference float64 floor decision for near-integer indices
            double ue = exact_u(ps, a.dom, ax, kkx, kky, kkz, hx, hy, hz, ax == 0 ? hx : (ax == 1 ? hy : hz));
            double fe = floor(ue);
            fl[ax] = (T)fe;
            f[ax] = (T)(ue - fe);
          }
        }
      }
      const cx<T> phk = ph;
      ph = ph * step;
      int ix = (int)fl[0], iy = (int)fl[1], iz = (int)fl[2];
      if (WRAP) {
        ix = ix < 0 ? ix + w0 : (ix >= w0 ? ix - w0 : ix);
        iy = iy < 0 ? iy + w1 : (iy >= w1 ? iy - w1 : iy);
        iz = iz < 0 ? iz + w2 : (iz >= w2 ? iz - w2 : iz);
      } else if ((unsigned)(ix + 1) > (unsigned)w0 || (unsigned)(iy + 1) > (unsigned)w1 ||
                 (unsigned)(iz + 1) > (unsigned)w2) {
        continue;  // whole footprint outside the window: exact zero contribution
      }
      const cx<T> base = C1[c1off] * phk;
      const P4* ptr = C2 + ((ix + 1) * (int)sx + (iy + 1) * (int)sy + (iz + 1));
      P4 e00 = ldg_pair(ptr), e10 = ldg_pair(ptr + sx), e01 = ldg_pair(ptr + sy), e11 = ldg_pair(ptr + sx + sy);
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
      cx<T> X0 = base * dU, X1 = base * dV, X2 = base * dS;
      rS += bV;
      axpy(rJ, j, bV);
      rX[0] += X0; rX[1] += X1; rX[2] += X2;
      axpy(rXJ[0], j, X0); axpy(rXJ[1], j, X1); axpy(rXJ[2], j, X2);
    }
    // fold the run: sum_j kappa_a(j) Y = kappa0_a sum Y + e_r,a sum j Y
    const T k0x = (T)kap[0], k0y = (T)kap[1], k0z = (T)kap[2];
    T* v = acc.v;
    v[0] += rS.re; v[1] += rS.im;
    v[2] += k0x * rS.re + er0 * rJ.re; v[3] += k0x * rS.im + er0 * rJ.im;
    v[4] += k0y * rS.re + er1 * rJ.re; v[5] += k0y * rS.im + er1 * rJ.im;
    v[6] += k0z * rS.re + er2 * rJ.re; v[7] += k0z * rS.im + er2 * rJ.im;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      v[8 + 6 * b] += k0x * rX[b].re + er0 * rXJ[b].re;  v[9 + 6 * b] += k0x * rX[b].im + er0 * rXJ[b].im;
      v[10 + 6 * b] += k0y * rX[b].re + er1 * rXJ[b].re; v[11 + 6 * b] += k0y * rX[b].im + er1 * rXJ[b].im;
      v[12 + 6 * b] += k0z * rX[b].re + er2 * rXJ[b].re; v[13 + 6 * b] += k0z * rX[b].im + er2 * rXJ[b].im;
    }
  }
  };
  if (tmask) unit_loop(std::true_type{});
  else unit_loop(std::false_type{});

  {
    const T* v = acc.v;
#pragma unroll
    for (int c = 0; c < kNumMoments; ++c) {
      T s = warp_sum(v[c]);
      if (lane == 0) wsum[warp][c] = (double)s;
    }
    __syncthreads();
    if (tid < kNumMoments) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) s += wsum[w][tid];
      red[tid] = s;
    }
    __syncthreads();
  }

  double* out = a.out + pose * 14;
  if (bpp == 1) {
    finalize(a, ps, red, out);
    return;
  }
  double* part = a.partials + (pose * bpp + blk) * kNumMoments;
  if (tid < kNumMoments) part[tid] = red[tid];
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(a.counters + pose, 1u);
  __syncthreads();
  if (ticket != (unsigned)(bpp - 1)) return;
  __threadfence();
  const double* pb = a.partials + pose * bpp * kNumMoments;
  for (int c = warp; c < kNumMoments; c += kWarps) {
    double s = 0.0;
    for (int b = lane; b < bpp; b += 32) s += __ldcg(pb + (int64_t)b * kNumMoments + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[c] = s;
  }
  __syncthreads();
  finalize(a, ps, red, out);
  if (tid == 0) a.counters[pose] = 0u;  // re-arm for the next launch
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
  if (grid > sm_count() * 16) grid = sm_count() * 16;
  if (precision == 32)
    pack_window_kernel<float><<<grid, 256, 0, st>>>((const cx<float>*)raw, (float4*)packed, w[0], w[1], w[2], wrap);
  else
    pack_window_kernel<double><<<grid, 256, 0, st>>>((const cx<double>*)raw, (double4*)packed, w[0], w[1], w[2], wrap);
  return cudaGetLastError();
}

cudaError_t launch_narrow(const void* src, void* dst, int64_t n, cudaStream_t st) {
  int grid = (int)ceil_div(n, 256);
  if (grid > sm_count() * 16) grid = sm_count() * 16;
  narrow_kernel<float><<<grid, 256, 0, st>>>((const cx<double>*)src, (cx<float>*)dst, n);
  return cudaGetLastError();
}

void plan_cascade(CascadeArgs& a, int64_t n_poses, int target_blocks) {
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

  if (n_poses == 1) {
    a.single = 1;
    a.blocks_per_pose = single_blocks(a, target_blocks);
    return;
  }
  a.single = 0;
  // direct gather: 16 x 16 mode patches x runs of L along the run axis
  // many poses: one run spans the whole run axis (fewer run folds and phase
  // restarts, measured +12 % at w = 96 over L = 8); few poses: short runs so
  // a pose splits over enough CTAs
  int L = a.seg_len > 0 ? a.seg_len : (n_poses >= target_blocks / 2 ? 1 << 30 : 4);
  int wmax = a.w[0] > a.w[1] ? a.w[0] : a.w[1];
  if (a.w[2] > wmax) wmax = a.w[2];
  if (a.dim == 2) L = 1;
  if (L > wmax) L = wmax;
  a.seg_len = L;
  // units per pose depend on the pose's run axis; bound by the worst case
  int64_t units = 1;
  {
    int64_t best = 0;
    for (int r = 0; r < 3; ++r) {
      int o1 = (r + 1) % 3, o2 = (r + 2) % 3;
      int64_t u = ceil_div(a.w[o1], 16) * ceil_div(a.w[o2], 16) * ceil_div(a.w[r], L);
      if (best == 0 || u < best) best = u;
    }
    units = best;
  }
  int64_t bpp = 1;
  if (n_poses < target_blocks) bpp = ceil_div(target_blocks, n_poses);
  if (bpp > units) bpp = units;
  if (bpp < 1) bpp = 1;
  a.blocks_per_pose = (int)bpp;
}

cudaError_t launch_cascade(const CascadeArgs& a, int64_t n_poses, cudaStream_t st) {
  if (a.single && n_poses == 1) return launch_cascade_single(a, st);
  // grid.x = poses x blocks_per_pose, issued in chunks that fit gridDim.x
  const int64_t max_blocks = (int64_t)1 << 30;
  int64_t chunk = max_blocks / a.blocks_per_pose;
  for (int64_t p0 = 0; p0 < n_poses; p0 += chunk) {
    int64_t np = n_poses - p0 < chunk ? n_poses - p0 : chunk;
    CascadeArgs c = a;
    c.pose_offset = a.pose_offset + p0;
    unsigned grid = (unsigned)(np * a.blocks_per_pose);
    const size_t tsm = (a.precision == 32 ? sizeof(cx<float>) : sizeof(cx<double>)) * (a.w[0] + a.w[1] + a.w[2]);
    if (a.precision == 32) {
      if (a.wrap) cascade3d_kernel<float, true><<<grid, kThreads, tsm, st>>>(c);
      else cascade3d_kernel<float, false><<<grid, kThreads, tsm, st>>>(c);
    } else {
      if (a.wrap) cascade3d_kernel<double, true><<<grid, kThreads, tsm, st>>>(c);
      else cascade3d_kernel<double, false><<<grid, kThreads, tsm, st>>>(c);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace gf
