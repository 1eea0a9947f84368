// cascade_tiled.cu -- u-space tiled cascade kernel (Q1 single query / Q3 sweep).
//
// Same semantics as cascade.cu (reference: _core.cascade_3d,
// /root/reference/pkg/src/geofield/_core.pyx:598-724); different data path.
//
// The gather of the moving window C2 at rotated continuous indices is the
// bottleneck of a direct implementation: neighbouring modes land in
// unrelated 128-byte lines, so every corner load costs one L1 wavefront per
// lane (profiles/r01_cascade_direct.md: LSU wavefronts 91% of peak).  This
// kernel inverts the loop.  C2's index space is cut into TS^3 cell tiles; a
// CTA stages one tile plus a one-cell halo on each side in shared memory
// (zero outside a truncated window, periodic for full spectra) and then
// enumerates exactly the modes k whose floor(u(k)) falls in that tile:
//
//   * for every (kx, ky) column of the tile's preimage the kz interval is
//     solved from the three slab constraints (conservatively widened), the
//     column intervals are prefix-summed across the block and expanded into
//     a shared-memory mode list;
//   * each candidate recomputes its canonical index u = fma(kz, Mz, base),
//     base = (T)(h + M[:,0] kx + M[:,1] ky) in float64, and is kept only if
//     floor(u) lies in the tile -- every mode has exactly one owner tile, so
//     the tiles partition the window exactly;
//   * the 8 corners are shared-memory loads; the reference's float64 floor
//     tie-break may move a corner by one cell, which the halo absorbs.
//
// Translation phase: per-axis tables px, py, pz (sincospi of float64-
// reduced arguments) per pose; a column carries px*py.  Moments and the
// fixed-order reductions are those of cascade.cu.
#include "cascade.cuh"
#include "common.cuh"

#include <math.h>

namespace gf {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <typename T> struct ColEntry {
  T base[3];     // canonical u offset of the column (u = fma(kz_k, Mz, base))
  int c1off;     // (kx * w1 + ky) * w2
  int kxy;       // kx | ky << 16
  cx<T> pxy;     // px[kx] * py[ky]
  T kapx, kapy;  // kx - hx, ky - hy
};

template <typename T> struct Tables {
  double mu[3][3];
  double R[9];
  double targ[3];
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// exclusive block scan of one int per thread; returns the block total
__device__ __forceinline__ int block_scan(int v, int* wtot, int& excl) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtot[warp] = x;
  __syncthreads();
  int before = 0, total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    int t = wtot[w];
    if (w < warp) before += t;
    total += t;
  }
  excl = before + x - v;
  __syncthreads();
  return total;
}

__device__ __forceinline__ double exact_u_t(const double* R, const double* dom, int a, int kx, int ky, int kz,
                                            int hx, int hy, int hz, int ha) {
  double ox = __dmul_rn((double)(kx - hx), dom[0]);
  double oy = __dmul_rn((double)(ky - hy), dom[1]);
  double oz = __dmul_rn((double)(kz - hz), dom[2]);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(R[0 + a], ox), __dmul_rn(R[3 + a], oy)), __dmul_rn(R[6 + a], oz));
  return __dadd_rn(__ddiv_rn(-s, dom[a]), (double)ha);
}

__device__ void finalize_out(const CascadeArgs& a, const double* R, const double* m, double* out) {
  const double TWO_PI = 6.283185307179586;
  double dc = a.dcell;
  out[0] = dc * m[0];
  out[1] = dc * m[1];
  for (int ax = 0; ax < 3; ++ax) {
    double k = dc * TWO_PI * a.dom[ax];
    out[2 + 2 * ax] = -k * m[3 + 2 * ax];
    out[3 + 2 * ax] = k * m[2 + 2 * ax];
  }
  double A[3][3][3] = {};
  for (int b = 0; b < 3; ++b) {
    A[0][1][b] = -R[6 + b]; A[0][2][b] = R[3 + b];
    A[1][0][b] = R[6 + b];  A[1][2][b] = -R[0 + b];
    A[2][0][b] = -R[3 + b]; A[2][1][b] = R[0 + b];
  }
  for (int g = 0; g < 3; ++g) {
    double gr = 0.0, gi = 0.0;
    for (int b = 0; b < 3; ++b)
      for (int ax = 0; ax < 3; ++ax) {
        double coef = -A[g][ax][b] * (a.dom[ax] / a.dom[b]);
        gr += coef * m[8 + 2 * (3 * b + ax)];
        gi += coef * m[9 + 2 * (3 * b + ax)];
      }
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

// shared-memory carve-up (dynamic): tile | coltab | list | px py pz
template <typename T, int TS> struct Smem {
  static constexpr int TP = TS + 3;                 // tile side incl. halo
  static constexpr int kTile = TP * TP * TP;        // cells
  static constexpr int kListCap = 16 * kThreads;    // mode-list entries per round
  static constexpr size_t tile_bytes = sizeof(cx<T>) * kTile;
  static constexpr size_t col_bytes = sizeof(ColEntry<T>) * kThreads;
  static constexpr size_t list_bytes = sizeof(unsigned) * kListCap;
  static constexpr size_t fixed = tile_bytes + col_bytes + list_bytes;
  static size_t total(const int w[3]) { return fixed + sizeof(cx<T>) * (w[0] + w[1] + w[2]); }
};

template <typename T, int TS>
__global__ void __launch_bounds__(kThreads, 2) cascade3d_tiled_kernel(CascadeArgs a) {
  using S = Smem<T, TS>;
  constexpr int TP = S::TP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cx<T>* tile = reinterpret_cast<cx<T>*>(smem_raw);
  ColEntry<T>* coltab = reinterpret_cast<ColEntry<T>*>(smem_raw + S::tile_bytes);
  unsigned* list = reinterpret_cast<unsigned*>(smem_raw + S::tile_bytes + S::col_bytes);
  cx<T>* ptab = reinterpret_cast<cx<T>*>(smem_raw + S::tile_bytes + S::col_bytes + S::list_bytes);

  __shared__ Tables<T> tb;
  __shared__ double minv[3][3];  // kappa = minv (u - h): minv[a][b] = -R[a][b] dw_b / dw_a
  __shared__ int wtot[kWarps];
  __shared__ double wsum[kWarps][kNumMoments];
  __shared__ double red[kNumMoments];
  __shared__ unsigned ticket;

  const int bpp = a.blocks_per_pose;
  const int64_t pose = a.pose_offset + blockIdx.x / bpp;
  const int blk = blockIdx.x % bpp;
  const int tid = threadIdx.x;
  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  const int wv[3] = {w0, w1, w2};

  // ---- per-pose constants and phase tables
  {
    const double* src = a.poses ? a.poses + pose * 12 : a.pose_inline;
    if (tid < 9) {
      tb.R[tid] = src[tid];
      int ia = tid / 3, ib = tid % 3;
      tb.mu[ia][ib] = -src[ib * 3 + ia] * (a.dom[ib] / a.dom[ia]);
    }
    if (tid >= 16 && tid < 19) tb.targ[tid - 16] = a.dom[tid - 16] * src[9 + tid - 16];
    if (tid >= 32 && tid < 41) {
      int ia = (tid - 32) / 3, ib = (tid - 32) % 3;
      minv[ia][ib] = -src[ia * 3 + ib] * (a.dom[ib] / a.dom[ia]);
    }
    __syncthreads();
    for (int i = tid; i < w0 + w1 + w2; i += kThreads) {
      int ax = i < w0 ? 0 : (i < w0 + w1 ? 1 : 2);
      int k = i - (ax == 0 ? 0 : (ax == 1 ? w0 : w0 + w1));
      int hh = ax == 0 ? hx : (ax == 1 ? hy : hz);
      double cyc = tb.targ[ax] * (double)(k - hh);
      cyc -= rint(cyc);
      T sn, cs;
      if constexpr (sizeof(T) == 4) sincospif(2.0f * (float)cyc, &sn, &cs);
      else sincospi(2.0 * cyc, &sn, &cs);
      ptab[i] = mk<T>(cs, sn);
    }
  }
  const cx<T>* px = ptab;
  const cx<T>* py = ptab + w0;
  const cx<T>* pz = ptab + w0 + w1;
  const T Mz[3] = {(T)tb.mu[0][2], (T)tb.mu[1][2], (T)tb.mu[2][2]};
  const T eps = (T)a.tie_eps;
  const cx<T>* __restrict__ C1 = reinterpret_cast<const cx<T>*>(a.C1);
  const cx<T>* __restrict__ C2 = reinterpret_cast<const cx<T>*>(a.C2p);  // raw window

  // tile grid over owner cells: non-wrap floor(u) in [-1, w-1], wrap [0, w)
  const int org = a.wrap ? 0 : -1;
  int ntile[3];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) ntile[ax] = (int)ceil_div(wv[ax] + (a.wrap ? 0 : 1), TS);
  const int tiles = ntile[0] * ntile[1] * ntile[2];

  Acc26<T> acc;
  acc.zero();
  __syncthreads();

  for (int tix = blk; tix < tiles; tix += bpp) {
    const int tz = tix % ntile[2], ty = (tix / ntile[2]) % ntile[1], tx = tix / (ntile[2] * ntile[1]);
    const int c0[3] = {org + TS * tx, org + TS * ty, org + TS * tz};
    // images (wrap): shifts n in {-1,0,1}^3 whose shifted tile meets the u range
    int nlo[3], nhi[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (!a.wrap) { nlo[ax] = nhi[ax] = 0; continue; }
      double span = fabs(tb.mu[ax][0]) * (hx + 1) + fabs(tb.mu[ax][1]) * (hy + 1) + fabs(tb.mu[ax][2]) * (hz + 1);
      double ulo = wv[ax] / 2 - span, uhi = wv[ax] / 2 + span;
      nlo[ax] = (int)floor((ulo - (c0[ax] + TS)) / wv[ax]);
      nhi[ax] = (int)ceil((uhi - c0[ax]) / wv[ax]);
    }
    bool loaded = false;
    for (int nx = nlo[0]; nx <= nhi[0]; ++nx)
      for (int ny = nlo[1]; ny <= nhi[1]; ++ny)
        for (int nz = nlo[2]; nz <= nhi[2]; ++nz) {
          const double cl[3] = {(double)(c0[0] + nx * w0), (double)(c0[1] + ny * w1), (double)(c0[2] + nz * w2)};
          // preimage bounding box of the cell box [cl, cl + TS] in kappa space
          double klo[3] = {1e30, 1e30, 1e30}, khi[3] = {-1e30, -1e30, -1e30};
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            double du[3] = {cl[0] + ((c & 1) ? TS : 0) - hx, cl[1] + ((c & 2) ? TS : 0) - hy,
                            cl[2] + ((c & 4) ? TS : 0) - hz};
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              double k = minv[i][0] * du[0] + minv[i][1] * du[1] + minv[i][2] * du[2];
              klo[i] = fmin(klo[i], k);
              khi[i] = fmax(khi[i], k);
            }
          }
          int kx0 = max((int)floor(klo[0]) - 1 + hx, 0), kx1 = min((int)ceil(khi[0]) + 1 + hx, w0 - 1);
          int ky0 = max((int)floor(klo[1]) - 1 + hy, 0), ky1 = min((int)ceil(khi[1]) + 1 + hy, w1 - 1);
          int kz0 = max((int)floor(klo[2]) - 1 + hz, 0), kz1 = min((int)ceil(khi[2]) + 1 + hz, w2 - 1);
          if (kx0 > kx1 || ky0 > ky1 || kz0 > kz1) continue;

          if (!loaded) {  // stage the tile (+ halo) once per tile
            __syncthreads();
            for (int e = tid; e < TP * TP * TP; e += kThreads) {
              int k = e % TP, j = (e / TP) % TP, i = e / (TP * TP);
              int gi = c0[0] - 1 + i, gj = c0[1] - 1 + j, gk = c0[2] - 1 + k;
              cx<T> v = mk<T>(0, 0);
              if (a.wrap) {
                gi = ((gi % w0) + w0) % w0; gj = ((gj % w1) + w1) % w1; gk = ((gk % w2) + w2) % w2;
                v = C2[((int64_t)gi * w1 + gj) * w2 + gk];
              } else if (gi >= 0 && gi < w0 && gj >= 0 && gj < w1 && gk >= 0 && gk < w2) {
                v = C2[((int64_t)gi * w1 + gj) * w2 + gk];
              }
              tile[e] = v;
            }
            loaded = true;
          }
          const T clT[3] = {(T)cl[0], (T)cl[1], (T)cl[2]};
          // owner cells of this tile: [c0, min(c0 + TS, w) - 1] (+ the image shift)
          const T clTe[3] = {(T)(cl[0] + min(TS, w0 - c0[0]) - 1), (T)(cl[1] + min(TS, w1 - c0[1]) - 1),
                             (T)(cl[2] + min(TS, w2 - c0[2]) - 1)};
          const int ncy = ky1 - ky0 + 1;
          const int ncols = (kx1 - kx0 + 1) * ncy;
          for (int cbase = 0; cbase < ncols; cbase += kThreads) {
            // ---- column pass: kz interval of this thread's column
            const int col = cbase + tid;
            int cnt = 0, zlo = 0;
            if (col < ncols) {
              const int kx = kx0 + col / ncy, ky = ky0 + col % ncy;
              const double kapx = kx - hx, kapy = ky - hy;
              double b3[3];
              double zl = kz0 - hz, zh = kz1 - hz;
#pragma unroll
              for (int ax = 0; ax < 3; ++ax) {
                b3[ax] = (double)(ax == 0 ? hx : (ax == 1 ? hy : hz)) + tb.mu[ax][0] * kapx + tb.mu[ax][1] * kapy;
                double m = tb.mu[ax][2];
                double lo = cl[ax] - b3[ax], hi = cl[ax] + TS - b3[ax];
                if (fabs(m) > 1e-12) {
                  double z1 = lo / m, z2 = hi / m;
                  zl = fmax(zl, fmin(z1, z2) - 1.0);
                  zh = fmin(zh, fmax(z1, z2) + 1.0);
                } else if (lo > 1.0 || hi < -1.0) {
                  zh = zl - 1.0;  // column never meets this slab
                }
              }
              if (zh >= zl) {
                int z0 = (int)ceil(zl) + hz, z1 = (int)floor(zh) + hz;
                z0 = max(z0, 0);
                z1 = min(z1, w2 - 1);
                if (z1 >= z0) {
                  cnt = z1 - z0 + 1;
                  zlo = z0;
                }
              }
              ColEntry<T> ce;
              ce.base[0] = (T)b3[0]; ce.base[1] = (T)b3[1]; ce.base[2] = (T)b3[2];
              ce.c1off = (kx * w1 + ky) * w2;
              ce.kxy = kx | (ky << 16);
              ce.pxy = px[kx] * py[ky];
              ce.kapx = (T)kapx; ce.kapy = (T)kapy;
              coltab[tid] = ce;
            }
            int off = 0;
            const int total = block_scan(cnt, wtot, off);
            for (int r0 = 0; r0 < total; r0 += S::kListCap) {
              // ---- expand this round's slice of the mode list
              for (int j = 0; j < cnt; ++j) {
                int pos = off + j - r0;
                if (pos >= 0 && pos < S::kListCap) list[pos] = ((unsigned)tid << 16) | (unsigned)(zlo + j);
              }
              __syncthreads();
              const int nr = min(total - r0, S::kListCap);
              for (int i = tid; i < nr; i += kThreads) {
                const unsigned e = list[i];
                const ColEntry<T>& ce = coltab[e >> 16];
                const int kz = (int)(e & 0xffffu);
                const T kapz = (T)(kz - hz);
                T u[3], fl[3], f[3];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                  u[ax] = fma(kapz, Mz[ax], ce.base[ax]);
                  fl[ax] = floor(u[ax]);
                }
                // ownership: floor(u) inside this (image of the) tile
                if (fl[0] < clT[0] || fl[0] > clTe[0] || fl[1] < clT[1] || fl[1] > clTe[1] || fl[2] < clT[2] ||
                    fl[2] > clTe[2])
                  continue;
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) f[ax] = u[ax] - fl[ax];
                const bool tz2 = a.dim == 3 && (f[2] < eps || f[2] > (T)1 - eps);
                if (f[0] < eps || f[0] > (T)1 - eps || f[1] < eps || f[1] > (T)1 - eps || tz2) {
                  const int kx = ce.kxy & 0xffff, ky = ce.kxy >> 16;
#pragma unroll
                  for (int ax = 0; ax < 3; ++ax) {
                    if ((ax < 2 || tz2) && (f[ax] < eps || f[ax] > (T)1 - eps)) {
                      double ue = exact_u_t(tb.R, a.dom, ax, kx, ky, kz, hx, hy, hz,
                                            ax == 0 ? hx : (ax == 1 ? hy : hz));
                      double fe = floor(ue);  // same image as the fast index, +-1 cell
                      fl[ax] = (T)fe;
                      f[ax] = (T)(ue - fe);
                    }
                  }
                }
                const int li = (int)(fl[0] - clT[0]) + 1, lj = (int)(fl[1] - clT[1]) + 1,
                          lk = (int)(fl[2] - clT[2]) + 1;
                const cx<T>* q = tile + (li * TP + lj) * TP + lk;
                const cx<T> c000 = q[0], c001 = q[1], c010 = q[TP], c011 = q[TP + 1];
                const cx<T> c100 = q[TP * TP], c101 = q[TP * TP + 1], c110 = q[TP * TP + TP],
                            c111 = q[TP * TP + TP + 1];
                const T fu = f[0], fv = f[1], fs = f[2];
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
                const cx<T> base = C1[ce.c1off + kz] * (ce.pxy * pz[kz]);
                cx<T> bV = base * V;
                cx<T> X0 = base * dU, X1 = base * dV, X2 = base * dS;
                acc.add(bV, X0, X1, X2, ce.kapx, ce.kapy, kapz);
              }
              __syncthreads();
            }
          }
        }
  }

  // ---- reductions (fixed order): warp -> block (float64) -> grid (last block)
  {
    const T* v = reinterpret_cast<const T*>(&acc);
    int lane = tid & 31, warp = tid >> 5;
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
    if (tid == 0) finalize_out(a, tb.R, red, out);
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
  const int lane = tid & 31, warp = tid >> 5;
  for (int c = warp; c < kNumMoments; c += kWarps) {
    double s = 0.0;
    for (int b = lane; b < bpp; b += 32) s += __ldcg(pb + (int64_t)b * kNumMoments + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) red[c] = s;
  }
  __syncthreads();
  if (tid == 0) {
    finalize_out(a, tb.R, red, out);
    a.counters[pose] = 0u;
  }
}

template <typename T, int TS>
cudaError_t launch_tiled_t(const CascadeArgs& a, int64_t n_poses, cudaStream_t st) {
  using S = Smem<T, TS>;
  const size_t smem = S::total(a.w);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(cascade3d_tiled_kernel<T, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int64_t max_blocks = (int64_t)1 << 30;
  int64_t chunk = max_blocks / a.blocks_per_pose;
  for (int64_t p0 = 0; p0 < n_poses; p0 += chunk) {
    int64_t np = n_poses - p0 < chunk ? n_poses - p0 : chunk;
    CascadeArgs c = a;
    c.pose_offset = a.pose_offset + p0;
    cascade3d_tiled_kernel<T, TS><<<(unsigned)(np * a.blocks_per_pose), kThreads, smem, st>>>(c);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

int tiled_tile_count(const CascadeArgs& a, int ts) {
  int n = 1;
  for (int ax = 0; ax < 3; ++ax) n *= (int)ceil_div(a.w[ax] + (a.wrap ? 0 : 1), ts);
  return n;
}

size_t tiled_smem_bytes(int precision, int ts, const int w[3]) {
  if (precision == 32) return ts == 16 ? Smem<float, 16>::total(w) : Smem<float, 8>::total(w);
  return Smem<double, 8>::total(w);
}

cudaError_t launch_cascade_tiled(const CascadeArgs& a, int64_t n_poses, cudaStream_t st) {
  if (a.precision == 32) {
    if (a.tile == 16) return launch_tiled_t<float, 16>(a, n_poses, st);
    return launch_tiled_t<float, 8>(a, n_poses, st);
  }
  return launch_tiled_t<double, 8>(a, n_poses, st);
}

}  // namespace gf
