// vector_torque.cu -- the moment-spectrum rotational gradient (SURVEY 8(f)#3:
// energy._rotational_gradient_vector, /root/reference/pkg/src/geofield/
// energy.py:210-251), the reference's independent cross-check of the torque.
//
// For every window mode w (float64 throughout, as the reference's numpy):
//   u = -R^T w / dw + h, V = multilinear sample of C2 at u, S_a the same of
//   the moving part's centre-referenced moment windows (rho p_a),
//   M_a = -S_a + c_a V, base = C1(w) exp(2 pi i w.t_eff),
//   G_g += base (sum_a (R^T Omega_g w)_a M_a + (w . Omega_g R c) V),
// and the result is 2 pi i dcell G_g for the d rotation generators Omega_g
// (_fallback.py:354-361).  One fused pass over the window: the four rotated
// samples share the corner indices and weights, nothing is materialised;
// block sums in a fixed-order tree, then one CTA sums the block partials in
// block order -- repeatable bit for bit.
#include "../../include/geofield_b200.h"
#include "common.cuh"

#include <math.h>

namespace gf {

int window_raw64(uint64_t h, const void** raw, int w[3], int* dim);  // capi.cu

namespace {

constexpr int kVT = 256;

struct VArgs {
  const cx<double>* C1;
  const cx<double>* W[4];  // C2, then the d moment windows
  int nwin;                // 1 + d
  int w[3];
  int wrap;
  double dom[3];
  double R[9];             // row-major, 2D embedded with R[2][2] = 1
  double teff[3];
  double c[3];
  double RtG[3][3][3];     // (R^T Omega_g)[a][b]
  double q[3][3];          // Omega_g R c
  int ngen;
  double* partials;        // nblocks x 6
};

__global__ void __launch_bounds__(kVT) vector_torque_kernel(VArgs a) {
  __shared__ double red[kVT / 32][6];
  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  const int64_t n = (int64_t)w0 * w1 * w2;
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t m = blockIdx.x * (int64_t)kVT + threadIdx.x; m < n; m += (int64_t)gridDim.x * kVT) {
    const int kz = (int)(m % w2);
    const int ky = (int)((m / w2) % w1);
    const int kx = (int)(m / ((int64_t)w1 * w2));
    const double om[3] = {(kx - hx) * a.dom[0], (ky - hy) * a.dom[1], (kz - hz) * a.dom[2]};
    int i0[3];
    double f[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // nu = -(W @ R); u = nu / dom + h (energy.py:230-231)
      const double nu = -__dadd_rn(__dadd_rn(__dmul_rn(om[0], a.R[0 + c]), __dmul_rn(om[1], a.R[3 + c])),
                                   __dmul_rn(om[2], a.R[6 + c]));
      const double u = __dadd_rn(__ddiv_rn(nu, a.dom[c]), (double)(c == 0 ? hx : (c == 1 ? hy : hz)));
      const double fl = floor(u);
      i0[c] = (int)fl;
      f[c] = u - fl;
    }
    cx<double> smp[4] = {mk<double>(0, 0), mk<double>(0, 0), mk<double>(0, 0), mk<double>(0, 0)};
#pragma unroll
    for (int corner = 0; corner < 8; ++corner) {
      const int d0 = corner >> 2, d1 = (corner >> 1) & 1, d2 = corner & 1;
      int ix = i0[0] + d0, iy = i0[1] + d1, iz = i0[2] + d2;
      if (a.wrap) {
        ix = ((ix % w0) + w0) % w0;
        iy = ((iy % w1) + w1) % w1;
        iz = ((iz % w2) + w2) % w2;
      } else if (ix < 0 || ix >= w0 || iy < 0 || iy >= w1 || iz < 0 || iz >= w2) {
        continue;  // zero outside a truncated window (_fallback.py:312-351)
      }
      const double wgt = (d0 ? f[0] : 1.0 - f[0]) * (d1 ? f[1] : 1.0 - f[1]) * (d2 ? f[2] : 1.0 - f[2]);
      const int64_t lin = ((int64_t)ix * w1 + iy) * w2 + iz;
      for (int k = 0; k < a.nwin; ++k) {
        const cx<double> v = a.W[k][lin];
        smp[k].re = fma(wgt, v.re, smp[k].re);
        smp[k].im = fma(wgt, v.im, smp[k].im);
      }
    }
    const cx<double> V = smp[0];
    double cyc = om[0] * a.teff[0] + om[1] * a.teff[1] + om[2] * a.teff[2];
    cyc -= rint(cyc);
    double sn, cs;
    sincospi(2.0 * cyc, &sn, &cs);
    const cx<double> base = a.C1[m] * mk<double>(cs, sn);
    cx<double> M[3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
      M[k] = k + 1 < a.nwin ? mk<double>(a.c[k] * V.re - smp[k + 1].re, a.c[k] * V.im - smp[k + 1].im)
                            : mk<double>(0, 0);
    for (int g = 0; g < a.ngen; ++g) {
      cx<double> s = mk<double>(0, 0);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double dir = a.RtG[g][k][0] * om[0] + a.RtG[g][k][1] * om[1] + a.RtG[g][k][2] * om[2];
        s.re = fma(dir, M[k].re, s.re);
        s.im = fma(dir, M[k].im, s.im);
      }
      const double lever = om[0] * a.q[g][0] + om[1] * a.q[g][1] + om[2] * a.q[g][2];
      s.re = fma(lever, V.re, s.re);
      s.im = fma(lever, V.im, s.im);
      const cx<double> t = base * s;
      acc[2 * g] += t.re;
      acc[2 * g + 1] += t.im;
    }
  }
  // fixed-order block sum: warp tree, then warps in order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double v = 0.0;
    for (int i = 0; i < kVT / 32; ++i) v += red[i][threadIdx.x];
    a.partials[(int64_t)blockIdx.x * 6 + threadIdx.x] = v;
  }
}

__global__ void sum_partials_kernel(const double* partials, int nblocks, double* out) {
  if (threadIdx.x < 6) {
    double v = 0.0;
    for (int b = 0; b < nblocks; ++b) v += partials[(int64_t)b * 6 + threadIdx.x];
    out[threadIdx.x] = v;
  }
}

}  // namespace
}  // namespace gf

using namespace gf;

extern "C" int gf_vector_torque(uint64_t h1, uint64_t h2, const uint64_t* hmom, int wrap, const double* domega,
                                double dcell, const double* R, const double* t_eff, const double* center,
                                double* out) {
  GF_CHECK(hmom && domega && R && t_eff && center && out, GF_EINVAL, "null argument");
  VArgs a = {};
  int w[3], d = 0;
  const void* p = nullptr;
  int rc = window_raw64(h1, &p, a.w, &d);
  if (rc) return rc;
  a.C1 = reinterpret_cast<const cx<double>*>(p);
  a.nwin = 1 + d;
  for (int k = 0; k < a.nwin; ++k) {
    int dk = 0;
    rc = window_raw64(k == 0 ? h2 : hmom[k - 1], &p, w, &dk);
    if (rc) return rc;
    GF_CHECK(dk == d && w[0] == a.w[0] && w[1] == a.w[1] && w[2] == a.w[2], GF_EINVAL, "window shape mismatch");
    a.W[k] = reinterpret_cast<const cx<double>*>(p);
  }
  a.wrap = wrap ? 1 : 0;
  double Rf[9];
  if (d == 3) {
    for (int k = 0; k < 9; ++k) Rf[k] = R[k];
  } else {
    const double e[9] = {R[0], R[1], 0.0, R[2], R[3], 0.0, 0.0, 0.0, 1.0};
    for (int k = 0; k < 9; ++k) Rf[k] = e[k];
  }
  for (int k = 0; k < 9; ++k) a.R[k] = Rf[k];
  for (int k = 0; k < 3; ++k) {
    a.dom[k] = k < d ? domega[k] : 1.0;
    a.teff[k] = k < d ? t_eff[k] : 0.0;
    a.c[k] = k < d ? center[k] : 0.0;
  }
  // generators (_fallback.py:354-361): about x, y, z in 3D; z alone in 2D
  const double G3[3][9] = {{0, 0, 0, 0, 0, -1, 0, 1, 0}, {0, 0, 1, 0, 0, 0, -1, 0, 0}, {0, -1, 0, 1, 0, 0, 0, 0, 0}};
  a.ngen = d == 3 ? 3 : 1;
  for (int g = 0; g < a.ngen; ++g) {
    const double* G = d == 3 ? G3[g] : G3[2];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double s = 0.0;  // (R^T G)[i][j] = sum_k R[k][i] G[k][j]
        for (int k = 0; k < 3; ++k) s += Rf[k * 3 + i] * G[k * 3 + j];
        a.RtG[g][i][j] = s;
      }
    double Rc[3];
    for (int i = 0; i < 3; ++i) Rc[i] = Rf[i * 3] * a.c[0] + Rf[i * 3 + 1] * a.c[1] + Rf[i * 3 + 2] * a.c[2];
    for (int i = 0; i < 3; ++i) a.q[g][i] = G[i * 3] * Rc[0] + G[i * 3 + 1] * Rc[1] + G[i * 3 + 2] * Rc[2];
  }
  const int64_t n = (int64_t)a.w[0] * a.w[1] * a.w[2];
  int nblocks = (int)ceil_div(n, kVT);
  if (nblocks > sm_count() * 8) nblocks = sm_count() * 8;
  void* buf = nullptr;
  cudaStream_t st = 0;
  GF_CUDA(cudaMallocAsync(&buf, sizeof(double) * (6 * (size_t)nblocks + 6), st));
  a.partials = reinterpret_cast<double*>(buf);
  vector_torque_kernel<<<nblocks, kVT, 0, st>>>(a);
  sum_partials_kernel<<<1, 32, 0, st>>>(a.partials, nblocks, a.partials + 6 * (size_t)nblocks);
  double sums[6];
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(sums, a.partials + 6 * (size_t)nblocks, sizeof sums, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(buf, st);
  GF_CUDA(e);
  // 2 pi i dcell G_g
  const double k = 6.283185307179586 * dcell;
  for (int g = 0; g < a.ngen; ++g) {
    out[2 * g] = -k * sums[2 * g + 1];
    out[2 * g + 1] = k * sums[2 * g];
  }
  for (int g = a.ngen; g < 3; ++g) out[2 * g] = out[2 * g + 1] = 0.0;
  return 0;
}
