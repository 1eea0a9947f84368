// field.cu -- full translational landscape (stage 4, F1/F2) and the rotated
// spectrum resampler.
//
// Reference: energy.score_field (/root/reference/pkg/src/geofield/
// energy.py:309-344) forms Q(w) = C1(w) V(w) exp(2 pi i w.(Rc - c)), with V
// the multilinear sample of C2 at u = -R^T w / dw + w/2
// (_fallback._interp_window, _fallback.py:312-351), embeds Q in the full
// DC-centred grid, multiplies by the origin phases and inverse-FFTs, / dV.
//
// Here the product kernel evaluates Q straight into the window (one thread
// per retained mode; same continuous index and float64 floor tie-break as
// the cascade kernels), with the origin phase folded into the same
// separable phase, and three pruned inverse passes (fft.cu) expand the w^d
// window to the N^d landscape with scale dcell = 1 / (N^d dV).  The same
// product kernel with C1 = 1 gives rotate_reflect_spectrum
// (spectral.py:204-226).
#include "../../include/geofield_b200.h"
#include "cascade.cuh"
#include "common.cuh"
#include "fft_core.cuh"

#include <math.h>
#include <stdlib.h>

extern "C" int gf_fft_pass(int precision, const void* in, void* out, const int32_t* shape_in,
                           const int32_t* shape_out, int axis, int n, int in_centered, int out_centered, int sign,
                           double in_phase, double out_phase, double scale, void* stream);

namespace gf {

// window handle internals (capi.cu)
int window_operands(uint64_t h1, uint64_t h2, int wrap, int precision, cudaStream_t st, const void** c1_raw,
                    const void** c2_packed, int w[3], int* dim);

namespace {

struct RotArgs {
  const void* C1;  // raw window (null: C1 = 1)
  const void* C2p; // packed moving window
  int w[3];
  int dim;
  double dom[3];
  double R[9];
  double s[3];     // phase exp(2 pi i w.s)
  double tie_eps;
  int kx0, nkx;    // window x-planes [kx0, kx0 + nkx) (slab decomposition)
  void* out;       // (nkx, w1, w2) complex<T>
  double mu[3][3];       // u_a = h_a + sum_b mu[a][b] kappa_b
  long long ufix[3][3];  // to_fix32(mu)
  int perm[3];           // brick lane order: fastest, middle, slowest mode axis
  int tie_dep[3];        // column a of R has one nonzero, in row tie_dep[a] (else -1)
};

__device__ __forceinline__ double exact_u_f(const double* R, const double* dom, int a, int kx, int ky, int kz, int hx,
                                            int hy, int hz, int ha) {
  double ox = __dmul_rn((double)(kx - hx), dom[0]);
  double oy = __dmul_rn((double)(ky - hy), dom[1]);
  double oz = __dmul_rn((double)(kz - hz), dom[2]);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(R[0 + a], ox), __dmul_rn(R[3 + a], oy)), __dmul_rn(R[6 + a], oz));
  return __dadd_rn(__ddiv_rn(-s, dom[a]), (double)ha);
}

// ---------------------------------------------------------------------------
// Brick-ordered product kernel: each CTA owns an 8 x 8 x 8 brick of window
// modes (2 per thread), so the rotated footprint of a CTA in C2 is a compact
// rotated brick -- each C2 sector comes from DRAM about once even when the
// packed window (2.2 GB at 512^3) is far larger than L2.  The gather is
// L1-wavefront bound, so lanes are laid out along the mode axes whose steps
// move least across C2's 128-byte rows: the fastest lane axis (`perm[0]`) is
// the mode axis with the largest component along C2's contiguous axis.  The
// gathered V * phase goes through shared memory and the C1 read and Q write
// are done in z-fastest order, coalesced.  fp32 indices in 32.32 fixed point.
// fp32: at most 51 registers so five CTAs (40 warps) share an SM -- the
// gathers are latency bound: 3.33 -> 3.16 ms for the 512^3 landscape against
// the default four (profiles/r02_product_occupancy.txt)
template <typename T, bool WRAP>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? 5 : 4) product_brick_kernel(RotArgs a) {
  using P4 = typename pair4<T>::type;
  __shared__ cx<T> sq[8 * 73];
  __shared__ cx<T> ph[3][8];  // exp(2 pi i dw_a s_a (k_a - h_a)) for this brick's 8 modes per axis
  __shared__ cx<T> tt[3][8];  // lattice-aligned poses: (floor, frac) of u_c at this brick's k_b, b = tie_dep[c]
  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  // brick (bx, by, bz) straight from a 3-D grid (z fastest): no index divisions
  const int bz = blockIdx.x, by = blockIdx.y, bx = blockIdx.z;
  const int t = threadIdx.x;
  const int sy = w2 + 1, sx = (w1 + 2) * (w2 + 1);
  const P4* __restrict__ C2 = reinterpret_cast<const P4*>(a.C2p);
  const cx<T>* __restrict__ C1 = reinterpret_cast<const cx<T>*>(a.C1);
  cx<T>* __restrict__ out = reinterpret_cast<cx<T>*>(a.out);
  const T eps = (T)a.tie_eps;
  const int pf = a.perm[0], pm = a.perm[1];
  if (t < 24) {  // float64 argument reduction, as the reference's per-axis phase (energy.py:339-341)
    const int ax = t >> 3, o = t & 7;
    const int k = ax == 0 ? a.kx0 + bx * 8 + o : (ax == 1 ? by * 8 + o : bz * 8 + o);
    const int h = ax == 0 ? hx : (ax == 1 ? hy : hz);
    double cyc = a.dom[ax] * a.s[ax] * (double)(k - h);
    cyc -= rint(cyc);
    double sn, cs;
    sincospi(2.0 * cyc, &sn, &cs);
    ph[ax][o] = mk<T>((T)cs, (T)sn);
  } else if (t >= 32 && t < 56) {  // tie table: row b, brick offset o
    const int b = (t - 32) >> 3, o = t & 7;
    const int k = b == 0 ? a.kx0 + bx * 8 + o : (b == 1 ? by * 8 + o : bz * 8 + o);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (a.tie_dep[c] != b) continue;
      const double ue = exact_u_f(a.R, a.dom, c, b == 0 ? k : hx, b == 1 ? k : hy, b == 2 ? k : hz, hx, hy, hz,
                                  c == 0 ? hx : (c == 1 ? hy : hz));
      const double fe = floor(ue);
      tt[b][o] = mk<T>((T)fe, (T)(ue - fe));
    }
  }
  __syncthreads();
  // C1 for the epilogue's (z-fastest) modes, issued before the gathers
  // brick origin in the (kx0-offset) C1 / output arrays, then 32-bit offsets
  const int64_t brick0 = ((int64_t)(bx * 8) * w1 + by * 8) * w2 + bz * 8;
  const int64_t c1brick0 = brick0 + (int64_t)a.kx0 * w1 * w2;
  const int plane = w1 * w2;
  cx<T> c1v[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int oz = t & 7, oy = (t >> 3) & 7, ox = (t >> 6) + 4 * h;
    const int kxl = bx * 8 + ox, ky = by * 8 + oy, kz = bz * 8 + oz;
    c1v[h] = mk<T>(1, 0);
    if (a.C1 && kxl < a.nkx && ky < w1 && kz < w2) c1v[h] = C1[c1brick0 + (ox * plane + oy * w2 + oz)];
  }
  // fp32 indices: the 32.32 fixed-point u of this thread's first mode, the
  // second (4 further along the slowest lane axis) by one exact 64-bit add
  long long u0[3] = {0, 0, 0};
  if constexpr (sizeof(T) == 4) {
    const int o_f = t & 7, o_m = (t >> 3) & 7, o_s = t >> 6;
    const int ox = pf == 0 ? o_f : (pm == 0 ? o_m : o_s);
    const int oy = pf == 1 ? o_f : (pm == 1 ? o_m : o_s);
    const int oz = pf == 2 ? o_f : (pm == 2 ? o_m : o_s);
    const int kk[3] = {a.kx0 + bx * 8 + ox - hx, by * 8 + oy - hy, bz * 8 + oz - hz};
#pragma unroll
    for (int ax = 0; ax < 3; ++ax)
      if ((ax < 2 || a.dim == 3 ? a.tie_dep[ax] : -1) < 0)  // the axes the loop below reads from u
        u0[ax] = ((long long)(ax == 0 ? hx : (ax == 1 ? hy : hz)) << 32) + (long long)kk[0] * a.ufix[ax][0] +
                 (long long)kk[1] * a.ufix[ax][1] + (long long)kk[2] * a.ufix[ax][2];
  }
  const int ps = 3 - pf - pm;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o_f = t & 7, o_m = (t >> 3) & 7, o_s = (t >> 6) + 4 * h;
    const int ox = pf == 0 ? o_f : (pm == 0 ? o_m : o_s);
    const int oy = pf == 1 ? o_f : (pm == 1 ? o_m : o_s);
    const int oz = pf == 2 ? o_f : (pm == 2 ? o_m : o_s);
    const int kxl = bx * 8 + ox, ky = by * 8 + oy, kz = bz * 8 + oz;
    if (kxl >= a.nkx || ky >= w1 || kz >= w2) continue;
    const int kx = a.kx0 + kxl;
    const int kk[3] = {kx - hx, ky - hy, kz - hz};
    T fl[3], f[3];
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        const int dep = ax < 2 || a.dim == 3 ? a.tie_dep[ax] : -1;
        if (dep >= 0) {  // lattice-aligned axis: tabulated reference floor / frac
          const cx<T> e = tt[dep][dep == 0 ? ox : (dep == 1 ? oy : oz)];
          fl[ax] = e.re;
          f[ax] = e.im;
          continue;
        }
        const long long u = u0[ax] + (h ? 4 * a.ufix[ax][ps] : 0);
        const unsigned lo = fix_lo(u);
        fl[ax] = (T)fix_floor(u);
        f[ax] = fix_frac(lo);
        if ((ax < 2 || a.dim == 3) && fix_tie(lo)) {
          double ue = exact_u_f(a.R, a.dom, ax, kx, ky, kz, hx, hy, hz, ax == 0 ? hx : (ax == 1 ? hy : hz));
          double fe = floor(ue);
          fl[ax] = (T)fe;
          f[ax] = (T)(ue - fe);
        }
      }
    } else {
#pragma unroll
      for (int ax = 0; ax < 3; ++ax) {
        double h0 = ax == 0 ? hx : (ax == 1 ? hy : hz);
        double u = h0 + a.mu[ax][0] * kk[0] + a.mu[ax][1] * kk[1] + a.mu[ax][2] * kk[2];
        fl[ax] = floor(u);
        f[ax] = u - fl[ax];
        if (!(ax < 2 || a.dim == 3)) continue;
        const int dep = a.tie_dep[ax];
        if (dep >= 0) {
          const cx<T> e = tt[dep][dep == 0 ? ox : (dep == 1 ? oy : oz)];
          fl[ax] = e.re;
          f[ax] = e.im;
        } else if (f[ax] < eps || f[ax] > (T)1 - eps) {
          double ue = exact_u_f(a.R, a.dom, ax, kx, ky, kz, hx, hy, hz, (int)h0);
          double fe = floor(ue);
          fl[ax] = fe;
          f[ax] = ue - fe;
        }
      }
    }
    int ix = (int)fl[0], iy = (int)fl[1], iz = (int)fl[2];
    cx<T> V = mk<T>(0, 0);
    bool live = true;
    if (WRAP) {
      ix = ix < 0 ? ix + w0 : (ix >= w0 ? ix - w0 : ix);
      iy = iy < 0 ? iy + w1 : (iy >= w1 ? iy - w1 : iy);
      iz = iz < 0 ? iz + w2 : (iz >= w2 ? iz - w2 : iz);
    } else if ((unsigned)(ix + 1) > (unsigned)w0 || (unsigned)(iy + 1) > (unsigned)w1 ||
               (unsigned)(iz + 1) > (unsigned)w2) {
      live = false;
    }
    if (live) {
      const P4* p = C2 + ((ix + 1) * sx + (iy + 1) * sy + (iz + 1));
      P4 e00 = ldg_pair(p), e10 = ldg_pair(p + sx), e01 = ldg_pair(p + sy), e11 = ldg_pair(p + sx + sy);
      const T fu = f[0], fv = f[1], fs = f[2];
      cx<T> a00 = lerp(mk<T>(e00.x, e00.y), mk<T>(e10.x, e10.y), fu);
      cx<T> a01 = lerp(mk<T>(e00.z, e00.w), mk<T>(e10.z, e10.w), fu);
      cx<T> a10 = lerp(mk<T>(e01.x, e01.y), mk<T>(e11.x, e11.y), fu);
      cx<T> a11 = lerp(mk<T>(e01.z, e01.w), mk<T>(e11.z, e11.w), fu);
      V = lerp(lerp(a00, a10, fv), lerp(a01, a11, fv), fs);
    }
    sq[ox * 73 + oy * 9 + oz] = V * ((ph[0][ox] * ph[1][oy]) * ph[2][oz]);
  }
  __syncthreads();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int oz = t & 7, oy = (t >> 3) & 7, ox = (t >> 6) + 4 * h;
    const int kxl = bx * 8 + ox, ky = by * 8 + oy, kz = bz * 8 + oz;
    if (kxl >= a.nkx || ky >= w1 || kz >= w2) continue;
    const cx<T> q = c1v[h] * sq[ox * 73 + oy * 9 + oz];
    out[brick0 + (ox * plane + oy * w2 + oz)] = q;
  }
}

}  // namespace
}  // namespace gf

using namespace gf;

extern "C" {

int gf_rotate_product_planes(uint64_t h1, uint64_t h2, int wrap, const double* domega, const double* R,
                             const double* s, int precision, int kx0, int nkx, void* out_dev, void* stream) {
  GF_CHECK(domega && R && s && out_dev, GF_EINVAL, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  RotArgs a = {};
  int rc = window_operands(h1, h2, wrap, precision, st, &a.C1, &a.C2p, a.w, &a.dim);
  if (rc) return rc;
  if (nkx < 0) {
    kx0 = 0;
    nkx = a.w[0];
  }
  GF_CHECK(kx0 >= 0 && kx0 + nkx <= a.w[0], GF_EINVAL, "plane range outside the window");
  a.kx0 = kx0;
  a.nkx = nkx;
  if (nkx == 0) return 0;
  for (int k = 0; k < 3; ++k) {
    a.dom[k] = k < a.dim ? domega[k] : 1.0;
    a.s[k] = k < a.dim ? s[k] : 0.0;
  }
  if (a.dim == 3) {
    for (int k = 0; k < 9; ++k) a.R[k] = R[k];
  } else {
    const double e[9] = {R[0], R[1], 0.0, R[2], R[3], 0.0, 0.0, 0.0, 1.0};
    for (int k = 0; k < 9; ++k) a.R[k] = e[k];
  }
  double umax = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    double v = a.w[ax] / 2;
    for (int b = 0; b < 3; ++b) v += (a.dom[b] / a.dom[ax]) * (a.w[b] / 2 + 1);
    umax = v > umax ? v : umax;
  }
  double eps = 8.0 * ldexp(umax, precision == 32 ? -23 : -52);
  double floor_eps = precision == 32 ? 1e-4 : 1e-9;
  a.tie_eps = eps > floor_eps ? eps : floor_eps;
  a.out = out_dev;
  for (int i = 0; i < 3; ++i)
    for (int jj = 0; jj < 3; ++jj) {
      a.mu[i][jj] = -a.R[jj * 3 + i] * (a.dom[jj] / a.dom[i]);
      a.ufix[i][jj] = to_fix32(a.mu[i][jj]);
    }
  for (int c = 0; c < 3; ++c) {
    const int nz = (a.R[c] != 0.0) + (a.R[3 + c] != 0.0) + (a.R[6 + c] != 0.0);
    a.tie_dep[c] = nz != 1 ? -1 : (a.R[c] != 0.0 ? 0 : (a.R[3 + c] != 0.0 ? 1 : 2));
  }
  // lane order: fastest along the mode axis whose u-step is most aligned with
  // C2's contiguous (z) axis, then the one most aligned with y
  {
    int pf = 0;
    for (int b = 1; b < 3; ++b)
      if (fabs(a.mu[2][b]) > fabs(a.mu[2][pf])) pf = b;
    int c0 = (pf + 1) % 3, c1 = (pf + 2) % 3;
    int pm = fabs(a.mu[1][c0]) >= fabs(a.mu[1][c1]) ? c0 : c1;
    a.perm[0] = pf;
    a.perm[1] = pm;
    a.perm[2] = 3 - pf - pm;
  }
  const dim3 bricks((unsigned)ceil_div(a.w[2], 8), (unsigned)ceil_div(a.w[1], 8), (unsigned)ceil_div(a.nkx, 8));
  GF_CHECK(bricks.y <= 65535 && bricks.z <= 65535, GF_EINVAL, "window too large for the brick grid");
  if (precision == 32) {
    if (wrap) product_brick_kernel<float, true><<<bricks, 256, 0, st>>>(a);
    else product_brick_kernel<float, false><<<bricks, 256, 0, st>>>(a);
  } else {
    if (wrap) product_brick_kernel<double, true><<<bricks, 256, 0, st>>>(a);
    else product_brick_kernel<double, false><<<bricks, 256, 0, st>>>(a);
  }
  GF_CUDA(cudaGetLastError());
  return 0;
}

int gf_rotate_product(uint64_t h1, uint64_t h2, int wrap, const double* domega, const double* R, const double* s,
                      int precision, void* out_dev, void* stream) {
  return gf_rotate_product_planes(h1, h2, wrap, domega, R, s, precision, 0, -1, out_dev, stream);
}

int gf_score_field(uint64_t h1, uint64_t h2, int wrap, const double* domega, const int32_t* dims, const double* R,
                   const double* s, double scale, int precision, void* work_dev, void* work2_dev, void* out_dev,
                   void* stream) {
  GF_CHECK(dims && work_dev && work2_dev && out_dev, GF_EINVAL, "null argument");
  const void* c1;
  const void* c2;
  int w[3], dim;
  int rc = window_operands(h1, h2, wrap, precision, (cudaStream_t)stream, &c1, &c2, w, &dim);
  if (rc) return rc;
  rc = gf_rotate_product(h1, h2, wrap, domega, R, s, precision, work_dev, stream);
  if (rc) return rc;
  // three pruned inverse passes: window-centred in, node order out
  int32_t N[3] = {dim == 3 ? dims[0] : 1, dim == 3 ? dims[1] : dims[0], dim == 3 ? dims[2] : dims[1]};
  int32_t W[3] = {dim == 3 ? w[0] : 1, dim == 3 ? w[1] : w[0], dim == 3 ? w[2] : w[1]};
  int32_t sh0[3] = {W[0], W[1], W[2]};
  int32_t sh1[3] = {W[0], W[1], N[2]};
  int32_t sh2[3] = {W[0], N[1], N[2]};
  int32_t sh3[3] = {N[0], N[1], N[2]};
  rc = gf_fft_pass(precision, work_dev, work2_dev, sh0, sh1, 2, N[2], 1, 0, 1, 0.0, 0.0, 1.0, stream);
  if (rc) return rc;
  if (dim == 3) {
    rc = gf_fft_pass(precision, work2_dev, work_dev, sh1, sh2, 1, N[1], 1, 0, 1, 0.0, 0.0, 1.0, stream);
    if (rc) return rc;
    rc = gf_fft_pass(precision, work_dev, out_dev, sh2, sh3, 0, N[0], 1, 0, 1, 0.0, 0.0, scale, stream);
  } else {
    rc = gf_fft_pass(precision, work2_dev, out_dev, sh1, sh2, 1, N[1], 1, 0, 1, 0.0, 0.0, scale, stream);
  }
  return rc;
}

}  // extern "C"
