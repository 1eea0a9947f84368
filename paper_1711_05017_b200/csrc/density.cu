// density.cu -- skeletal-density construction on the grid (stage 1, D1a-D2).
//
// Compiled with -fmad=false (see _build.py): every float64 product and sum is
// separately rounded, exactly as the reference's plain -O3 x86-64 build of
// _core.pyx, so point-element distances, exclusion (xi < eta_floor h),
// subdivision decisions, residual flags and occupancy reproduce the
// reference bit for bit.  Values agree to a few ulps, well inside the 1e-12
// the tests use: exp/atan2 differ from libm by ulps, and the 3D sweep leaf
// regroups its divisions and uses exp2 and explicit FMAs (sweep_kernel); no
// decision is taken on a regrouped quantity.
//
// Reference kernels (/root/reference/pkg/src/geofield/_core.pyx):
//   distance   _tri_dist_3d 65-99, distance_3d 189-230 (BVH; here a brute
//              min over all elements -- the min is order-independent, so the
//              value is identical), 2D 26-41/149-186
//   winding    _tri_solid_angle 244-259, winding_3d 277-292, 2D 237-274
//   sweep      sweep_3d 385-523 (4-way midpoint DFS, children pushed c0, c1,
//              c2, centre and popped LIFO), 2D 300-382
//   combine    descriptor.affinity_field 309-357, _neighbor_average 283-306
//
// GPU layout: one thread per grid node; elements staged through shared
// memory in tiles (coalesced, reused by the whole block); the sweep's DFS
// keeps one frame per level (triangle + next-child index) in local memory
// instead of the reference's 200-entry stack.
#include "../../include/geofield_b200.h"
#include "common.cuh"

#include <math.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <string.h>
#include <vector>

namespace gf {
namespace {

constexpr int kThreads = 128;
constexpr int kSweepThreads = 256;
constexpr int kTile = 128;  // elements per shared-memory tile

struct d3 { double x, y, z; };

__device__ __forceinline__ double seg_dist_2d(double ax, double ay, double bx, double by, double px, double py) {
  double dx = bx - ax, dy = by - ay;
  double den = dx * dx + dy * dy;
  double t = 0.0;
  if (den > 1e-300) {
    t = ((px - ax) * dx + (py - ay) * dy) / den;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  }
  double cx = ax + t * dx - px, cy = ay + t * dy - py;
  return sqrt(cx * cx + cy * cy);
}

__device__ __forceinline__ double seg_dist_3d(d3 a, d3 b, d3 p) {
  double dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
  double den = dx * dx + dy * dy + dz * dz;
  double t = 0.0;
  if (den > 1e-300) {
    t = ((p.x - a.x) * dx + (p.y - a.y) * dy + (p.z - a.z) * dz) / den;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  }
  double cx = a.x + t * dx - p.x, cy = a.y + t * dy - p.y, cz = a.z + t * dz - p.z;
  return sqrt(cx * cx + cy * cy + cz * cz);
}

__device__ __forceinline__ double tri_dist(d3 v0, d3 v1, d3 v2, d3 p) {
  double e0x = v1.x - v0.x, e0y = v1.y - v0.y, e0z = v1.z - v0.z;
  double e1x = v2.x - v0.x, e1y = v2.y - v0.y, e1z = v2.z - v0.z;
  double nx = e0y * e1z - e0z * e1y;
  double ny = e0z * e1x - e0x * e1z;
  double nz = e0x * e1y - e0y * e1x;
  double nn = sqrt(nx * nx + ny * ny + nz * nz);
  double dx = p.x - v0.x, dy = p.y - v0.y, dz = p.z - v0.z;
  double dot00 = e0x * e0x + e0y * e0y + e0z * e0z;
  double dot01 = e0x * e1x + e0y * e1y + e0z * e1z;
  double dot11 = e1x * e1x + e1y * e1y + e1z * e1z;
  double d0 = dx * e0x + dy * e0y + dz * e0z;
  double d1 = dx * e1x + dy * e1y + dz * e1z;
  double den = dot00 * dot11 - dot01 * dot01;
  if (den < 1e-300) den = 1e-300;
  double u = (dot11 * d0 - dot01 * d1) / den;
  double v = (dot00 * d1 - dot01 * d0) / den;
  if (u >= 0.0 && v >= 0.0 && u + v <= 1.0) {
    if (nn < 1e-300) nn = 1e-300;
    return fabs(dx * nx + dy * ny + dz * nz) / nn;
  }
  double m = seg_dist_3d(v0, v1, p);
  double s = seg_dist_3d(v1, v2, p);
  if (s < m) m = s;
  s = seg_dist_3d(v0, v2, p);
  if (s < m) m = s;
  return m;
}

__device__ __forceinline__ double solid_angle(d3 v0, d3 v1, d3 v2, d3 p) {
  double ax = v0.x - p.x, ay = v0.y - p.y, az = v0.z - p.z;
  double bx = v1.x - p.x, by = v1.y - p.y, bz = v1.z - p.z;
  double cx = v2.x - p.x, cy = v2.y - p.y, cz = v2.z - p.z;
  double la = sqrt(ax * ax + ay * ay + az * az);
  double lb = sqrt(bx * bx + by * by + bz * bz);
  double lc = sqrt(cx * cx + cy * cy + cz * cz);
  double num = ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz) + az * (bx * cy - by * cx);
  double den = la * lb * lc + (ax * bx + ay * by + az * bz) * lc + (ax * cx + ay * cy + az * cz) * lb +
               (bx * cx + by * cy + bz * cz) * la;
  return 2.0 * atan2(num, den);
}

// node coordinate origin + spacing * i (descriptor.py:141-146), unfused
__device__ __forceinline__ double node_coord(double o, double h, int i) { return o + h * (double)i; }

struct PointSource {
  const double* P;  // explicit points (m x d) or null -> grid nodes
  int d;
  int dims[3];
  double origin[3];
  double spacing;
  int x0;  // global index of local plane 0 along axis 0 (slab sharding)
  __device__ __forceinline__ void get(int64_t i, double* p) const {
    if (P) {
      for (int a = 0; a < d; ++a) p[a] = P[i * d + a];
      return;
    }
    if (d == 3) {
      int k = (int)(i % dims[2]);
      int64_t r = i / dims[2];
      int j = (int)(r % dims[1]);
      int ii = (int)(r / dims[1]);
      p[0] = node_coord(origin[0], spacing, ii + x0);
      p[1] = node_coord(origin[1], spacing, j);
      p[2] = node_coord(origin[2], spacing, k);
    } else {
      int j = (int)(i % dims[1]);
      int ii = (int)(i / dims[1]);
      p[0] = node_coord(origin[0], spacing, ii + x0);
      p[1] = node_coord(origin[1], spacing, j);
    }
  }
  // node visited by thread slot g: row-major, or (3D grid nodes whose (y, z)
  // plane tiles by BY x BZ) BY x BZ patches of one plane, so a block's nodes
  // are spatially compact and its culling decisions agree
  template <int BY, int BZ>
  __device__ __forceinline__ int64_t node_of(int64_t g) const {
    if (P || d != 3 || dims[1] % BY || dims[2] % BZ) return g;
    const int64_t pn = (int64_t)dims[1] * dims[2];
    const int64_t plane = g / pn;
    const int r = (int)(g - plane * pn);
    const int t = r % (BY * BZ), b = r / (BY * BZ);
    const int nbz = dims[2] / BZ;
    const int j = (b / nbz) * BY + t / BZ, k = (b % nbz) * BZ + t % BZ;
    return plane * pn + (int64_t)j * dims[2] + k;
  }
};

// ---------------------------------------------------------------------------
// D1a + D1b fused: exact min distance and winding number per point

template <int D>
__global__ void __launch_bounds__(kThreads) dist_wind_kernel(PointSource src, const double* __restrict__ elems,
                                                             int64_t ne, int64_t m, double* __restrict__ xi_out,
                                                             double* __restrict__ wind_out) {
  constexpr int E = D == 3 ? 9 : 4;
  __shared__ double tile[kTile * E];
  const int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  const bool live = i < m;
  double p[3] = {0.0, 0.0, 0.0};
  if (live) src.get(i, p);
  double best = 1e300, acc = 0.0;
  for (int64_t e0 = 0; e0 < ne; e0 += kTile) {
    const int n = (int)min((int64_t)kTile, ne - e0);
    __syncthreads();
    for (int t = threadIdx.x; t < n * E; t += kThreads) tile[t] = elems[e0 * E + t];
    __syncthreads();
    if (!live) continue;
    for (int e = 0; e < n; ++e) {
      const double* q = tile + e * E;
      if (D == 3) {
        d3 v0 = {q[0], q[1], q[2]}, v1 = {q[3], q[4], q[5]}, v2 = {q[6], q[7], q[8]}, pp = {p[0], p[1], p[2]};
        double dd = tri_dist(v0, v1, v2, pp);
        if (dd < best) best = dd;
        acc += solid_angle(v0, v1, v2, pp);
      } else {
        double dd = seg_dist_2d(q[0], q[1], q[2], q[3], p[0], p[1]);
        if (dd < best) best = dd;
        double ux = q[0] - p[0], uy = q[1] - p[1], vx = q[2] - p[0], vy = q[3] - p[1];
        acc += atan2(ux * vy - uy * vx, ux * vx + uy * vy);
      }
    }
  }
  if (live) {
    if (xi_out) xi_out[i] = best;
    if (wind_out) wind_out[i] = D == 3 ? acc / 12.566370614359172 : acc / 6.283185307179586;
  }
}

// ---------------------------------------------------------------------------
// D1a + D1b on grid nodes, culled (3D).  Same values and decisions as
// dist_wind_kernel, with less work per node:
//  * distance: the elements are also kept in a spatially sorted copy whose
//    tiles carry a bounding sphere (centre, inflated radius) and one of
//    their vertices.  A node's upper bound on its min distance is its
//    distance to the nearest such vertex (a point of the surface), lowered
//    to the running minimum as tiles are evaluated; a tile whose lower bound
//    |p - c_t| - r_t exceeds it (1e-9 relative + 1e-12 coordinate-scale
//    margin) cannot hold the minimum and is skipped.  The min is
//    order-independent, so the value is the same bits as the full loop
//    (the reference's BVH prunes the same way, _core.pyx:189-230).
//  * winding: with `wind_bbox`, a node outside the (closed) mesh's inflated
//    bounding box has winding number 0 up to rounding, so `inside` is false
//    exactly as in the reference; the sum is skipped and 0 stored.  Used
//    only where the winding value itself is not returned (the skeletal
//    family, where it decides occupancy alone).
// Tiles are loaded only when some node of the block needs them.
struct CullInfo {
  const double* sorted;    // ne x 9, spatially ordered copy of the elements
  const double4* spheres;  // per kTile tile of `sorted`: centre xyz, radius
  const double4* reps;     // per tile: one vertex of the tile (xyz)
  int ntiles;
  double scale;            // max(1, |coordinate|) over the elements
  int wind_bbox;           // 1: winding only for nodes inside [lo, hi]
  double lo[3], hi[3];
};

__global__ void __launch_bounds__(kThreads) dist_wind_culled_kernel(PointSource src, const double* __restrict__ elems,
                                                                    int64_t ne, int64_t m, CullInfo ci,
                                                                    double* __restrict__ xi_out,
                                                                    double* __restrict__ wind_out) {
  __shared__ double tile[kTile * 9];
  static_assert(kThreads == 16 * 8, "brick shape");
  const int64_t g = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  const bool live = g < m;
  const int64_t i = live ? src.node_of<16, 8>(g) : g;
  double p[3] = {0.0, 0.0, 0.0};
  if (live) src.get(i, p);
  const d3 pp = {p[0], p[1], p[2]};
  double best = 1e300;
  if (xi_out) {
    // upper bound of the min distance: the nearest tile vertex
    double ub2 = 1e300;
    for (int t = 0; t < ci.ntiles; ++t) {
      const double4 v = ci.reps[t];
      const double dx = p[0] - v.x, dy = p[1] - v.y, dz = p[2] - v.z;
      ub2 = fmin(ub2, dx * dx + dy * dy + dz * dz);
    }
    const double ub = sqrt(ub2);
    const double slack = 1e-12 * (fabs(p[0]) + fabs(p[1]) + fabs(p[2]) + ci.scale);
    for (int t = 0; t < ci.ntiles; ++t) {
      const double4 s = ci.spheres[t];
      const double dx = p[0] - s.x, dy = p[1] - s.y, dz = p[2] - s.z;
      const double bound = fmin(ub, best) * (1.0 + 1e-9) + slack;
      const bool need = live && sqrt(dx * dx + dy * dy + dz * dz) - s.w <= bound;
      if (!__syncthreads_or(need)) continue;
      const int64_t e0 = (int64_t)t * kTile;
      const int n = (int)min((int64_t)kTile, ne - e0);
      for (int k = threadIdx.x; k < n * 9; k += kThreads) tile[k] = ci.sorted[e0 * 9 + k];
      __syncthreads();
      if (need) {
        for (int e = 0; e < n; ++e) {
          const double* q = tile + e * 9;
          const double dd = tri_dist({q[0], q[1], q[2]}, {q[3], q[4], q[5]}, {q[6], q[7], q[8]}, pp);
          if (dd < best) best = dd;
        }
      }
      __syncthreads();
    }
  }
  if (wind_out) {
    const bool inb = p[0] >= ci.lo[0] && p[0] <= ci.hi[0] && p[1] >= ci.lo[1] && p[1] <= ci.hi[1] &&
                     p[2] >= ci.lo[2] && p[2] <= ci.hi[2];
    const bool need = live && (!ci.wind_bbox || inb);
    double acc = 0.0;
    if (__syncthreads_or(need)) {
      for (int64_t e0 = 0; e0 < ne; e0 += kTile) {  // original element order: the reference's summation order
        const int n = (int)min((int64_t)kTile, ne - e0);
        __syncthreads();
        for (int k = threadIdx.x; k < n * 9; k += kThreads) tile[k] = elems[e0 * 9 + k];
        __syncthreads();
        if (!need) continue;
        for (int e = 0; e < n; ++e) {
          const double* q = tile + e * 9;
          acc += solid_angle({q[0], q[1], q[2]}, {q[3], q[4], q[5]}, {q[6], q[7], q[8]}, pp);
        }
      }
    }
    if (live) wind_out[i] = need ? acc / 12.566370614359172 : 0.0;
  }
  if (live && xi_out) xi_out[i] = best;
}

// ---------------------------------------------------------------------------
// D1c: adaptive skeletal sweep

struct SweepParams {
  double sigma, gconst, max_angle, eta_min, ginv;
  int max_depth;
  double max_angle_lo;  // max_angle (1 - 1e-9): the margin of the depth-0 shortcut
};

// 1 / x to about an ulp for normal positive x: the MUFU seed and two Newton steps
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = __fma_rn(-x, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-x, r, 1.0);
  return __fma_rn(r, e, r);
}

// one leaf from its centroid offset m = centroid - p and eta = |m|.
// The reference's four divisions (dot area / eta, eta / xi, / sigma, / den)
// and its exp are regrouped: g = exp2(-(eta - xi)^2 gk) with
// gk = log2(e) / (2 (xi sigma)^2) per node, scale = gconst g dot area times a
// Newton reciprocal of eta den.  The terms move by a few ulps (the values are
// compared at 1e-12; every decision -- subdivision, residual, clamp,
// exact-zero skip -- is taken on unchanged quantities).
__device__ __forceinline__ void leaf_3d_c(double mx, double my, double mz, double eta, double area, double n0,
                                          double n1, double n2, double xi, double gk, const SweepParams& sp,
                                          double& re, double& im, int64_t& ncl) {
  if (eta < sp.eta_min) {
    eta = sp.eta_min;
    ++ncl;
  }
  // value arithmetic with explicit FMAs (this file is built -fmad=false for the decisions)
  const double dot = __fma_rn(mz, n2, __fma_rn(my, n1, mx * n0));
  const double dd = eta - xi;
  const double g = exp2(-(dd * dd) * gk) * sp.ginv;
  const double z2r = __fma_rn(-eta, eta, xi * xi);
  const double z2i = (2.0 * xi) * eta;
  const double den = __fma_rn(z2r, z2r, z2i * z2i);
  const double scale = sp.gconst * g * (dot * area) * rcp_nr(eta * den);
  re = __fma_rn(scale, z2r, re);
  im = __fma_rn(-scale, z2i, im);
}

__device__ __forceinline__ void leaf_3d(const d3& a, const d3& b, const d3& c, double area, const d3& p,
                                        const double* nrm, double xi, double gk, const SweepParams& sp, double& re,
                                        double& im, int64_t& ncl) {
  const double mx = (a.x + b.x + c.x) / 3.0 - p.x;
  const double my = (a.y + b.y + c.y) / 3.0 - p.y;
  const double mz = (a.z + b.z + c.z) / 3.0 - p.z;
  leaf_3d_c(mx, my, mz, sqrt(mx * mx + my * my + mz * mz), area, nrm[0], nrm[1], nrm[2], xi, gk, sp, re, im, ncl);
}

struct Tri { d3 a, b, c; };

// child k of a split triangle in the reference's pop order:
// k = 0 centre (m01, m12, m02), 1 corner2 (m02, m12, v2),
// 2 corner1 (m01, v1, m12), 3 corner0 (v0, m01, m02)   (_core.pyx:439-500)
__device__ __forceinline__ Tri child_tri(const Tri& P, int k) {
  d3 m01 = {0.5 * (P.a.x + P.b.x), 0.5 * (P.a.y + P.b.y), 0.5 * (P.a.z + P.b.z)};
  d3 m02 = {0.5 * (P.a.x + P.c.x), 0.5 * (P.a.y + P.c.y), 0.5 * (P.a.z + P.c.z)};
  d3 m12 = {0.5 * (P.b.x + P.c.x), 0.5 * (P.b.y + P.c.y), 0.5 * (P.b.z + P.c.z)};
  if (k == 0) return Tri{m01, m12, m02};
  if (k == 1) return Tri{m02, m12, P.c};
  if (k == 2) return Tri{m01, P.b, m12};
  return Tri{P.a, m01, m02};
}

// kSweepThreads nodes per CTA share every staged element tile (the kernel is
// bound by the L2 -> shared traffic of the tiles at ~10^5 elements).
// 3D tiles also carry each triangle's bounding radius about its centroid
// (`radii`, inflated): at depth 0, if area / (|p - centroid| - r)^2 is
// below max_angle (1e-9 margin), the reference's measure test
// area / (dist^2 + 1e-300) > max_angle cannot fire, so the exact distance is
// not needed -- the face is a leaf, with the same bits and no residual.
// Exact zeros (3D): a leaf whose centroid distance eta exceeds
// thr = xi (1 + 38.7 sigma) has |targ| > 38.7, exp(-targ^2 / 2) underflows to
// +0 and its terms are +-0, which leave re and im unchanged bit for bit; such
// a face is skipped after the depth-0 test, and a whole tile is skipped when
// its sphere (`tiles`: centre, radius, largest measure) puts every centroid
// beyond thr and every face through the depth-0 shortcut (no subdivision, no
// residual).  Element centroids are staged once per tile with the
// reference's expression ((a + b + c) / 3).
template <int D>
__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(PointSource src, const double* __restrict__ elems,
                                                              const double* __restrict__ normals,
                                                              const double* __restrict__ measures,
                                                              const double* __restrict__ radii,
                                                              const double* __restrict__ tiles, int64_t ne, int64_t m,
                                                              const double* __restrict__ xi_eff, SweepParams sp,
                                                              double* __restrict__ out, double* __restrict__ resid,
                                                              int64_t* __restrict__ clamps) {
  constexpr int E = D == 3 ? 9 : 4;
  // tile record: 3D [centroid 3 | radius | measure | normal 3 | vertices 9 | pad], 144 bytes, so the
  // depth-0 path reads its eight values as four 16-byte loads; 2D [segment 4 | normal 2 | measure]
  constexpr int ET = D == 3 ? 18 : 7;
  constexpr int OV = D == 3 ? 8 : 0, ON = D == 3 ? 5 : 4, OM = D == 3 ? 4 : 6;
  constexpr int kThreads = kSweepThreads;
  __shared__ __align__(16) double tile[kTile * ET];
  static_assert(kThreads == 16 * 16, "brick shape");
  const int64_t g = blockIdx.x * (int64_t)kThreads + threadIdx.x;
  const bool live = g < m;
  const int64_t i = live ? src.node_of<16, 16>(g) : g;
  double p3[3] = {0.0, 0.0, 0.0};
  if (live) src.get(i, p3);
  const d3 p = {p3[0], p3[1], p3[2]};
  const double xi = live ? xi_eff[i] : 1.0;
  double re = 0.0, im = 0.0, worst = live ? resid[i] : 0.0;
  int64_t ncl = 0;
  // DFS frames: the split ancestor at each level and how many of its
  // children have been handed out (replaces the reference's 200-entry stack)
  Tri frame[24];
  unsigned char taken[24];

  const double thr = xi * (1.0 + 38.7 * sp.sigma) * (1.0 + 1e-9);
  const double gk = 0.7213475204444817 / ((xi * sp.sigma) * (xi * sp.sigma));
  const double pslack = 1e-12 * (fabs(p.x) + fabs(p.y) + fabs(p.z));
  for (int64_t e0 = 0; e0 < ne; e0 += kTile) {
    const int n = (int)min((int64_t)kTile, ne - e0);
    bool need = live;
    if (D == 3 && need) {
      const double* ts = tiles + 5 * (e0 / kTile);
      const double dx = p.x - ts[0], dy = p.y - ts[1], dz = p.z - ts[2];
      const double lb = sqrt(dx * dx + dy * dy + dz * dz) - ts[3] - pslack;
      need = !(lb > thr && ts[4] < sp.max_angle_lo * (lb * lb));
    }
    if (!__syncthreads_or(need)) continue;
    for (int t = threadIdx.x; t < n * E; t += kThreads) tile[(t / E) * ET + OV + t % E] = elems[e0 * E + t];
    for (int t = threadIdx.x; t < n * D; t += kThreads) tile[(t / D) * ET + ON + t % D] = normals[e0 * D + t];
    for (int t = threadIdx.x; t < n; t += kThreads) tile[t * ET + OM] = measures[e0 + t];
    if (D == 3)
      for (int t = threadIdx.x; t < n; t += kThreads) {
        const double* g = elems + (e0 + t) * 9;
        double* o = tile + t * ET;
        o[0] = (g[0] + g[3] + g[6]) / 3.0;
        o[1] = (g[1] + g[4] + g[7]) / 3.0;
        o[2] = (g[2] + g[5] + g[8]) / 3.0;
        o[3] = radii[e0 + t];
      }
    __syncthreads();
    if (need) for (int e = 0; e < n; ++e) {
      const double* q = tile + e * ET;
      const double* nrm = q + ON;
      double meas = q[OM];
      int depth = 0;
      constexpr int nchild = D == 3 ? 4 : 2;
      Tri cur;
      if (D == 3) {  // far face: a depth-0 leaf without the exact distance (see above)
        const double2 c01 = *reinterpret_cast<const double2*>(q);
        const double2 c2r = *reinterpret_cast<const double2*>(q + 2);
        const double2 mn0 = *reinterpret_cast<const double2*>(q + 4);
        const double2 n12 = *reinterpret_cast<const double2*>(q + 6);
        const double mx = c01.x - p.x;
        const double my = c01.y - p.y;
        const double mz = c2r.x - p.z;
        const double eta = sqrt(mx * mx + my * my + mz * mz);
        const double lb = eta - c2r.y;
        if (lb > 0.0 && meas < sp.max_angle_lo * (lb * lb)) {
          if (eta > thr) continue;  // exact zero
          leaf_3d_c(mx, my, mz, eta, mn0.x, mn0.y, n12.x, n12.y, xi, gk, sp, re, im, ncl);
          continue;
        }
        const double* v = q + OV;
        cur = Tri{{v[0], v[1], v[2]}, {v[3], v[4], v[5]}, {v[6], v[7], v[8]}};
      } else {
        cur = Tri{{q[0], q[1], 0.0}, {q[2], q[3], 0.0}, {0.0, 0.0, 0.0}};
      }
      while (true) {
        double measure;
        if (D == 3) {
          double de = tri_dist(cur.a, cur.b, cur.c, p);
          measure = meas / (de * de + 1e-300);
        } else {
          double de = seg_dist_2d(cur.a.x, cur.a.y, cur.b.x, cur.b.y, p.x, p.y);
          if (de < 1e-300) de = 1e-300;
          measure = meas / de;
        }
        if (measure > sp.max_angle && depth < sp.max_depth) {
          frame[depth] = cur;
          taken[depth] = 1;
          if (D == 3) {
            cur = child_tri(cur, 0);
            meas = 0.25 * meas;
          } else {  // (m, b) is popped before (a, m)   (_core.pyx:344-361)
            cur = Tri{{0.5 * (cur.a.x + cur.b.x), 0.5 * (cur.a.y + cur.b.y), 0.0}, cur.b, cur.c};
            meas = 0.5 * meas;
          }
          ++depth;
          continue;
        }
        if (measure > sp.max_angle && measure > worst) worst = measure;
        if (D == 3) {
          leaf_3d(cur.a, cur.b, cur.c, meas, p, nrm, xi, gk, sp, re, im, ncl);
        } else {
          double mx = 0.5 * (cur.a.x + cur.b.x) - p.x, my = 0.5 * (cur.a.y + cur.b.y) - p.y;
          double eta = sqrt(mx * mx + my * my);
          if (eta < sp.eta_min) {
            eta = sp.eta_min;
            ++ncl;
          }
          double dot = mx * nrm[0] + my * nrm[1];
          double dA = dot * meas / eta;
          double targ = (eta / xi - 1.0) / sp.sigma;
          double g = exp(-0.5 * targ * targ) * sp.ginv;
          double z2r = xi * xi - eta * eta;
          double z2i = 2.0 * xi * eta;
          double den = z2r * z2r + z2i * z2i;
          double scale = sp.gconst * g * dA / den;
          re += scale * z2r;
          im -= scale * z2i;
        }
        // next pending sibling, climbing out of exhausted levels
        while (depth > 0 && taken[depth - 1] == nchild) {
          --depth;
          meas = D == 3 ? 4.0 * meas : 2.0 * meas;
        }
        if (depth == 0) break;
        const Tri& P = frame[depth - 1];
        if (D == 3) {
          cur = child_tri(P, taken[depth - 1]);
        } else {
          cur = Tri{P.a, {0.5 * (P.a.x + P.b.x), 0.5 * (P.a.y + P.b.y), 0.0}, P.c};
        }
        ++taken[depth - 1];
      }
    }
  }
  if (live) {
    out[2 * i] = re;
    out[2 * i + 1] = im;
    resid[i] = worst;
    clamps[i] += ncl;
  }
}

__global__ void clamp_min_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t m, double lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] > lo ? x[i] : lo;  // np.maximum(xi, eta_min)
}

// stats[0] = total clamps, stats[1] = worst residual (integer atomics only:
// the sum is exact and the max of non-negative doubles is order-free)
__global__ void stats_kernel(const double* __restrict__ resid, const int64_t* __restrict__ clamps, int64_t m,
                             unsigned long long* acc) {
  unsigned long long c = 0, w = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    c += (unsigned long long)clamps[i];
    unsigned long long b = (unsigned long long)__double_as_longlong(resid[i]);
    w = b > w ? b : w;
  }
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_down_sync(0xffffffffu, c, o);
    unsigned long long t = __shfl_down_sync(0xffffffffu, w, o);
    w = t > w ? t : w;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(acc, c);
    atomicMax(acc + 1, w);
  }
}

// ---------------------------------------------------------------------------
// D2: combine (inside ? lam_in conj(I+) : -lam_out I+), exclusion, flags

__global__ void combine_kernel(int64_t m, const double* __restrict__ xi, const double* __restrict__ wind,
                               const double* __restrict__ iplus, const double* __restrict__ resid, int family,
                               double lam_in, double lam_out, double eta_min, double max_angle,
                               double* __restrict__ values, uint8_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const bool inside = wind[i] >= 0.5;
    const bool excluded = xi[i] < eta_min;
    double vr, vi;
    if (family == 0) {  // InverseSquare: the winding number itself
      vr = wind[i];
      vi = 0.0;
    } else if (inside) {
      vr = lam_in * iplus[2 * i];
      vi = lam_in * -iplus[2 * i + 1];
    } else {
      vr = -lam_out * iplus[2 * i];
      vi = -lam_out * iplus[2 * i + 1];
    }
    values[2 * i] = vr;
    values[2 * i + 1] = vi;
    const bool unresolved = family != 0 && resid[i] > max_angle;
    // bit0 excluded, bit1 unresolved, bit2 inside
    flags[i] = (uint8_t)((excluded ? 1 : 0) | (unresolved ? 2 : 0) | (inside ? 4 : 0));
  }
}

// excluded nodes take the mean of their non-excluded face neighbours
// (descriptor.py:283-306): neighbours summed in the reference's order
// (axis 0 -1/+1 ... axis d-1), 0 when none.
__global__ void neighbor_fill_kernel(int d, int n0, int n1, int n2, const double* __restrict__ values,
                                     const uint8_t* __restrict__ flags, double* __restrict__ out) {
  const int64_t m = (int64_t)n0 * n1 * n2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    double vr = values[2 * i], vi = values[2 * i + 1];
    if (flags[i] & 1) {
      int c[3];
      int dims[3] = {n0, n1, n2};
      int64_t r = i;
      for (int a = d - 1; a >= 0; --a) {
        c[a] = (int)(r % dims[a]);
        r /= dims[a];
      }
      int64_t stride[3];
      stride[d - 1] = 1;
      for (int a = d - 2; a >= 0; --a) stride[a] = stride[a + 1] * dims[a + 1];
      double ar = 0.0, ai = 0.0;
      int cnt = 0;
      for (int a = 0; a < d; ++a) {
        // reference order: off = -1 (source c-1) then off = +1 (source c+1)
        for (int s = 0; s < 2; ++s) {
          int cc = s == 0 ? c[a] - 1 : c[a] + 1;
          if (cc < 0 || cc >= dims[a]) continue;
          int64_t j = i + (s == 0 ? -stride[a] : stride[a]);
          if (flags[j] & 1) continue;
          ar += values[2 * j];
          ai += values[2 * j + 1];
          ++cnt;
        }
      }
      if (cnt > 0) {
        vr = ar / (double)cnt;
        vi = ai / (double)cnt;
      } else {
        vr = 0.0;
        vi = 0.0;
      }
    }
    out[2 * i] = vr;
    out[2 * i + 1] = vi;
  }
}

}  // namespace
}  // namespace gf

using namespace gf;

namespace {

double __longlong_as_double_host(unsigned long long b) {
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
}

// Per-thread cache of device blocks for the per-call buffers: repeated
// fields of the same size reuse memory instead of paying cudaMalloc and the
// device-synchronising cudaFree every call.  Blocks go back to the cache
// when the entry point returns (after its final stream synchronisation).
struct BlockCache {
  std::multimap<size_t, void*> free_blocks;
  size_t cached = 0;
  ~BlockCache() {
    for (auto& kv : free_blocks) cudaFree(kv.second);  // process exit: errors ignored
  }
};
thread_local BlockCache tl_blocks;
constexpr size_t kBlockCacheCap = size_t(8) << 30;

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t alloc(size_t bytes) {
    auto it = tl_blocks.free_blocks.lower_bound(bytes);
    if (it != tl_blocks.free_blocks.end() && it->first <= 2 * bytes + (1 << 20)) {
      p = it->second;
      n = it->first;
      tl_blocks.cached -= n;
      tl_blocks.free_blocks.erase(it);
      return cudaSuccess;
    }
    n = bytes;
    return cudaMalloc(&p, bytes);
  }
  ~DevBuf() {
    if (!p) return;
    if (tl_blocks.cached + n > kBlockCacheCap) {
      gf::device_free(p);
      return;
    }
    tl_blocks.free_blocks.emplace(n, p);
    tl_blocks.cached += n;
  }
};

int upload(const void* host, size_t bytes, DevBuf& b, cudaStream_t st) {
  if (bytes == 0) return 0;
  GF_CUDA(b.alloc(bytes));
  GF_CUDA(cudaMemcpyAsync(b.p, host, bytes, cudaMemcpyHostToDevice, st));
  return 0;
}

int check_dim(int d) {
  GF_CHECK(d == 2 || d == 3, GF_EINVAL, "dimension must be 2 or 3");
  return 0;
}

// Sweep aids of a triangle set, both inflated so rounding can only make them
// larger: per-triangle bounding radius about the centroid (a + b + c) / 3
// (the depth-0 shortcut), and per kTile tile of the ORIGINAL element order
// (the sweep sums in that order) a bounding sphere of the tile's vertices
// plus its largest measure: {cx, cy, cz, r, max measure} (the zero-tile cull).
struct SweepAids {
  std::vector<double> radii, tiles;
};

SweepAids sweep_aids(const double* el, const double* meas, int64_t ne) {
  SweepAids s;
  s.radii.resize(ne);
  double scale = 1.0;
  for (int64_t k = 0; k < 9 * ne; ++k) scale = std::max(scale, std::fabs(el[k]));
  for (int64_t e = 0; e < ne; ++e) {
    const double* q = el + 9 * e;
    const double c[3] = {(q[0] + q[3] + q[6]) / 3.0, (q[1] + q[4] + q[7]) / 3.0, (q[2] + q[5] + q[8]) / 3.0};
    double m = 0.0;
    for (int v = 0; v < 3; ++v) {
      const double dx = q[3 * v] - c[0], dy = q[3 * v + 1] - c[1], dz = q[3 * v + 2] - c[2];
      m = std::max(m, std::sqrt(dx * dx + dy * dy + dz * dz));
    }
    s.radii[e] = m * (1.0 + 1e-12) + 1e-300;
  }
  const int64_t nt = ceil_div(ne, kTile);
  s.tiles.resize(5 * nt);
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t e1 = std::min(ne, (t + 1) * kTile);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300}, mx = 0.0;
    for (int64_t e = t * kTile; e < e1; ++e) {
      mx = std::max(mx, meas[e]);
      for (int k = 0; k < 9; ++k) {
        lo[k % 3] = std::min(lo[k % 3], el[9 * e + k]);
        hi[k % 3] = std::max(hi[k % 3], el[9 * e + k]);
      }
    }
    const double c[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    double r = 0.0;
    for (int64_t e = t * kTile; e < e1; ++e)
      for (int v = 0; v < 3; ++v) {
        const double* q = el + 9 * e + 3 * v;
        const double dx = q[0] - c[0], dy = q[1] - c[1], dz = q[2] - c[2];
        r = std::max(r, std::sqrt(dx * dx + dy * dy + dz * dz));
      }
    double* o = &s.tiles[5 * t];
    o[0] = c[0];
    o[1] = c[1];
    o[2] = c[2];
    o[3] = r * (1.0 + 1e-12) + 1e-12 * scale;
    o[4] = mx;
  }
  return s;
}

// Culling aids of a closed triangle set for dist_wind_culled_kernel: the
// elements in Morton order of their centroids (compact tiles), one inflated
// bounding sphere per tile, and the inflated bounding box.
struct CullHost {
  std::vector<double> sorted;
  std::vector<double4> spheres;  // ntiles spheres, then ntiles representative vertices
  double lo[3], hi[3], scale;
};

void build_cull(const double* el, int64_t ne, CullHost& h) {
  for (int a = 0; a < 3; ++a) {
    h.lo[a] = 1e300;
    h.hi[a] = -1e300;
  }
  for (int64_t v = 0; v < 3 * ne; ++v)  // every vertex of every triangle
    for (int a = 0; a < 3; ++a) {
      h.lo[a] = std::min(h.lo[a], el[3 * v + a]);
      h.hi[a] = std::max(h.hi[a], el[3 * v + a]);
    }
  double ext = 0.0;
  for (int a = 0; a < 3; ++a) ext = std::max(ext, h.hi[a] - h.lo[a]);
  std::vector<std::pair<uint32_t, int64_t>> key(ne);
  for (int64_t e = 0; e < ne; ++e) {
    const double* q = el + 9 * e;
    uint32_t code = 0;
    for (int a = 0; a < 3; ++a) {
      const double c = (q[a] + q[3 + a] + q[6 + a]) / 3.0;
      uint32_t v = (uint32_t)std::min(1023.0, std::max(0.0, (c - h.lo[a]) / (ext + 1e-300) * 1024.0));
      for (int b = 0; b < 10; ++b) code |= ((v >> b) & 1u) << (3 * b + a);
    }
    key[e] = {code, e};
  }
  std::stable_sort(key.begin(), key.end());
  h.sorted.resize(9 * ne);
  for (int64_t e = 0; e < ne; ++e) std::memcpy(&h.sorted[9 * e], el + 9 * key[e].second, 9 * sizeof(double));
  const int64_t nt = ceil_div(ne, kTile);
  h.spheres.resize(2 * nt);
  h.scale = 1.0;
  for (int64_t k = 0; k < 9 * ne; ++k) h.scale = std::max(h.scale, std::fabs(el[k]));
  for (int64_t t = 0; t < nt; ++t) {
    const double* v0 = &h.sorted[9 * t * kTile];
    h.spheres[nt + t] = make_double4(v0[0], v0[1], v0[2], 0.0);
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    const int64_t e1 = std::min(ne, (t + 1) * kTile);
    for (int64_t e = t * kTile; e < e1; ++e)
      for (int v = 0; v < 3; ++v)
        for (int a = 0; a < 3; ++a) {
          lo[a] = std::min(lo[a], h.sorted[9 * e + 3 * v + a]);
          hi[a] = std::max(hi[a], h.sorted[9 * e + 3 * v + a]);
        }
    const double c[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    double r = 0.0;
    for (int64_t e = t * kTile; e < e1; ++e)
      for (int v = 0; v < 3; ++v) {
        const double* q = &h.sorted[9 * e + 3 * v];
        const double dx = q[0] - c[0], dy = q[1] - c[1], dz = q[2] - c[2];
        r = std::max(r, std::sqrt(dx * dx + dy * dy + dz * dz));
      }
    h.spheres[t] = make_double4(c[0], c[1], c[2], r * (1.0 + 1e-12) + 1e-300);
  }
  for (int a = 0; a < 3; ++a) {
    const double pad = 1e-9 * (ext + std::fabs(h.lo[a]) + std::fabs(h.hi[a]));
    h.lo[a] -= pad;
    h.hi[a] += pad;
  }
}

// upload the culling aids; ci points into the device buffers
int upload_cull(const CullHost& h, int64_t ne, int wind_bbox, DevBuf& ds, DevBuf& dsp, CullInfo& ci,
                cudaStream_t st) {
  int rc = upload(h.sorted.data(), sizeof(double) * 9 * ne, ds, st);
  if (rc) return rc;
  if ((rc = upload(h.spheres.data(), sizeof(double4) * h.spheres.size(), dsp, st))) return rc;
  ci.sorted = (const double*)ds.p;
  ci.ntiles = (int)(h.spheres.size() / 2);
  ci.spheres = (const double4*)dsp.p;
  ci.reps = ci.spheres + ci.ntiles;
  ci.scale = h.scale;
  ci.wind_bbox = wind_bbox;
  for (int a = 0; a < 3; ++a) {
    ci.lo[a] = h.lo[a];
    ci.hi[a] = h.hi[a];
  }
  return 0;
}

}  // namespace

extern "C" {

int gf_distance_winding(int d, const double* elems, int64_t ne, const double* P, int64_t m, double* xi_out,
                        double* wind_out) {
  int rc = check_dim(d);
  if (rc) return rc;
  GF_CHECK(elems && P && (xi_out || wind_out) && ne > 0 && m >= 0, GF_EINVAL, "bad argument");
  if (m == 0) return 0;
  cudaStream_t st = 0;
  DevBuf de, dp, dx, dw;
  const int E = d == 3 ? 9 : 4;
  if ((rc = upload(elems, sizeof(double) * E * ne, de, st))) return rc;
  if ((rc = upload(P, sizeof(double) * d * m, dp, st))) return rc;
  if (xi_out) GF_CUDA(dx.alloc(sizeof(double) * m));
  if (wind_out) GF_CUDA(dw.alloc(sizeof(double) * m));
  PointSource src = {};
  src.P = (const double*)dp.p;
  src.d = d;
  unsigned grid = (unsigned)ceil_div(m, kThreads);
  DevBuf dsorted, dspheres;
  if (d == 3 && xi_out && !wind_out && m >= 256) {
    // distances only, many points: the tile-culled kernel (same bits: the
    // min is order-independent and the culling is conservative)
    CullHost ch;
    build_cull(elems, ne, ch);
    CullInfo ci;
    if ((rc = upload_cull(ch, ne, 0, dsorted, dspheres, ci, st))) return rc;
    dist_wind_culled_kernel<<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, ci, (double*)dx.p, nullptr);
    GF_CUDA(cudaStreamSynchronize(st));  // `ch` leaves scope
  } else if (d == 3) {
    dist_wind_kernel<3><<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, (double*)dx.p, (double*)dw.p);
  } else {
    dist_wind_kernel<2><<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, (double*)dx.p, (double*)dw.p);
  }
  GF_CUDA(cudaGetLastError());
  if (xi_out) GF_CUDA(cudaMemcpyAsync(xi_out, dx.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  if (wind_out) GF_CUDA(cudaMemcpyAsync(wind_out, dw.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int gf_winding_grid(int d, const double* elems, int64_t ne, const int32_t* dims, const double* origin, double spacing,
                    void* wind_dev, void* stream) {
  int rc = check_dim(d);
  if (rc) return rc;
  GF_CHECK(elems && dims && origin && wind_dev && ne > 0, GF_EINVAL, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t m = 1;
  for (int a = 0; a < d; ++a) m *= dims[a];
  DevBuf de, dx;
  const int E = d == 3 ? 9 : 4;
  if ((rc = upload(elems, sizeof(double) * E * ne, de, st))) return rc;
  PointSource src = {};
  src.P = nullptr;
  src.d = d;
  for (int a = 0; a < 3; ++a) {
    src.dims[a] = a < d ? dims[a] : 1;
    src.origin[a] = a < d ? origin[a] : 0.0;
  }
  src.spacing = spacing;
  unsigned grid = (unsigned)ceil_div(m, kThreads);
  if (d == 3) {  // winding only (the exact sum at every node: the indicator returns the value)
    CullInfo ci = {};
    dist_wind_culled_kernel<<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, ci, nullptr,
                                                       (double*)wind_dev);
  } else {
    GF_CUDA(dx.alloc(sizeof(double) * m));  // the 2D kernel writes distances too
  }
  if (d == 2)
    dist_wind_kernel<2><<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, (double*)dx.p, (double*)wind_dev);
  GF_CUDA(cudaGetLastError());
  GF_CUDA(cudaStreamSynchronize(st));  // the element and distance buffers go back to the cache
  return 0;
}

int gf_sweep(int d, const double* elems, const double* normals, const double* measures, int64_t ne, const double* P,
             const double* xi_eff, int64_t m, double sigma, double gconst, double max_angle, int max_depth,
             double eta_min, double* out_c128, double* resid, int64_t* clamps) {
  int rc = check_dim(d);
  if (rc) return rc;
  GF_CHECK(elems && normals && measures && P && xi_eff && out_c128 && resid && clamps && ne > 0, GF_EINVAL,
           "bad argument");
  GF_CHECK(max_depth >= 0 && max_depth <= 24, GF_EINVAL, "max_depth must be in [0, 24]");
  if (m == 0) return 0;
  cudaStream_t st = 0;
  const int E = d == 3 ? 9 : 4;
  DevBuf de, dn, dm, dp, dx, dout, dres, dcl;
  if ((rc = upload(elems, sizeof(double) * E * ne, de, st))) return rc;
  if ((rc = upload(normals, sizeof(double) * d * ne, dn, st))) return rc;
  if ((rc = upload(measures, sizeof(double) * ne, dm, st))) return rc;
  if ((rc = upload(P, sizeof(double) * d * m, dp, st))) return rc;
  if ((rc = upload(xi_eff, sizeof(double) * m, dx, st))) return rc;
  if ((rc = upload(resid, sizeof(double) * m, dres, st))) return rc;
  if ((rc = upload(clamps, sizeof(int64_t) * m, dcl, st))) return rc;
  GF_CUDA(dout.alloc(sizeof(double) * 2 * m));
  PointSource src = {};
  src.P = (const double*)dp.p;
  src.d = d;
  SweepParams sp = {sigma, gconst, max_angle, eta_min, 1.0 / (2.5066282746310002 * sigma), max_depth,
                      max_angle * (1.0 - 1e-9)};
  unsigned grid = (unsigned)ceil_div(m, kSweepThreads);
  DevBuf drad, dtil;
  if (d == 3) {
    const SweepAids aids = sweep_aids(elems, measures, ne);
    if ((rc = upload(aids.radii.data(), sizeof(double) * ne, drad, st))) return rc;
    if ((rc = upload(aids.tiles.data(), sizeof(double) * aids.tiles.size(), dtil, st))) return rc;
    sweep_kernel<3><<<grid, kSweepThreads, 0, st>>>(src, (const double*)de.p, (const double*)dn.p,
                                                    (const double*)dm.p, (const double*)drad.p,
                                                    (const double*)dtil.p, ne, m, (const double*)dx.p, sp,
                                                    (double*)dout.p, (double*)dres.p, (int64_t*)dcl.p);
    GF_CUDA(cudaStreamSynchronize(st));  // `aids` leaves scope
  } else {
    sweep_kernel<2><<<grid, kSweepThreads, 0, st>>>(src, (const double*)de.p, (const double*)dn.p,
                                                    (const double*)dm.p, nullptr, nullptr, ne, m,
                                                    (const double*)dx.p, sp, (double*)dout.p, (double*)dres.p,
                                                    (int64_t*)dcl.p);
  }
  GF_CUDA(cudaGetLastError());
  GF_CUDA(cudaMemcpyAsync(out_c128, dout.p, sizeof(double) * 2 * m, cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaMemcpyAsync(resid, dres.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaMemcpyAsync(clamps, dcl.p, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int gf_affinity_planes(int d, const double* elems, const double* normals, const double* measures, int64_t ne,
                       const int32_t* dims, const double* origin, double spacing, int32_t plane0, int32_t nplanes,
                       int32_t halo_lo, int32_t halo_hi, int family, double sigma, double gconst, double lam_in,
                       double lam_out, double max_angle, int max_depth, double eta_floor, void* values_dev,
                       uint8_t* flags_dev, double* stats, void* stream) {
  int rc = check_dim(d);
  if (rc) return rc;
  GF_CHECK(elems && normals && measures && dims && origin && values_dev && flags_dev && stats && ne > 0, GF_EINVAL,
           "bad argument");
  GF_CHECK(max_depth >= 0 && max_depth <= 24, GF_EINVAL, "max_depth must be in [0, 24]");
  GF_CHECK(nplanes > 0 && plane0 >= 0 && plane0 + nplanes <= dims[0], GF_EINVAL, "plane range outside the grid");
  GF_CHECK(halo_lo >= 0 && halo_hi >= 0 && plane0 - halo_lo >= 0 && plane0 + nplanes + halo_hi <= dims[0], GF_EINVAL,
           "halo outside the grid");
  cudaStream_t st = (cudaStream_t)stream;
  const int E = d == 3 ? 9 : 4;
  int64_t plane = 1;
  for (int a = 1; a < d; ++a) plane *= dims[a];
  const int lo = plane0 - halo_lo, cnt = nplanes + halo_lo + halo_hi;
  const int64_t m = (int64_t)cnt * plane;          // nodes computed (owned + halo planes)
  const int64_t own = (int64_t)nplanes * plane;    // nodes returned
  const int64_t off = (int64_t)halo_lo * plane;    // first owned node in the computed block
  const bool halos = halo_lo || halo_hi;
  DevBuf de, dn, dm, dxi, dwind, dxe, dip, dres, dcl, dval, hval, hflg;
  if ((rc = upload(elems, sizeof(double) * E * ne, de, st))) return rc;
  if ((rc = upload(normals, sizeof(double) * d * ne, dn, st))) return rc;
  if ((rc = upload(measures, sizeof(double) * ne, dm, st))) return rc;
  GF_CUDA(dxi.alloc(sizeof(double) * m));
  GF_CUDA(dwind.alloc(sizeof(double) * m));
  GF_CUDA(dres.alloc(sizeof(double) * m));
  GF_CUDA(dcl.alloc(sizeof(int64_t) * m));
  GF_CUDA(dip.alloc(sizeof(double) * 2 * m));
  GF_CUDA(dval.alloc(sizeof(double) * 2 * m));
  GF_CUDA(cudaMemsetAsync(dres.p, 0, sizeof(double) * m, st));
  GF_CUDA(cudaMemsetAsync(dcl.p, 0, sizeof(int64_t) * m, st));
  // with halo planes, fill a full computed block and hand back the owned part
  void* out_vals = values_dev;
  uint8_t* out_flags = flags_dev;
  if (halos) {
    GF_CUDA(hval.alloc(sizeof(double) * 2 * m));
    GF_CUDA(hflg.alloc(m));
    out_vals = hval.p;
    out_flags = (uint8_t*)hflg.p;
  }
  PointSource src = {};
  src.P = nullptr;
  src.d = d;
  for (int a = 0; a < 3; ++a) {
    src.dims[a] = a < d ? dims[a] : 1;
    src.origin[a] = a < d ? origin[a] : 0.0;
  }
  src.dims[0] = cnt;
  src.x0 = lo;
  src.spacing = spacing;
  const double eta_min = eta_floor * spacing;
  unsigned grid = (unsigned)ceil_div(m, kThreads);
  // per-stage device time for the stats (the reference reports seconds_*)
  cudaEvent_t ev[3];
  for (auto& e : ev) GF_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
    }
  } ev_guard{ev};
  GF_CUDA(cudaEventRecord(ev[0], st));
  DevBuf dsorted, dspheres, drad, dtil;
  SweepAids aids;  // (alive until the final synchronize)
  if (d == 3) {
    // winding values leave this pipeline only for the inverse-square family;
    // the skeletal family needs occupancy alone (the bounding-box shortcut)
    CullHost ch;
    build_cull(elems, ne, ch);
    CullInfo ci;
    if ((rc = upload_cull(ch, ne, family != 0 ? 1 : 0, dsorted, dspheres, ci, st))) return rc;
    dist_wind_culled_kernel<<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, ci, (double*)dxi.p,
                                                       (double*)dwind.p);
    aids = sweep_aids(elems, measures, ne);
    if ((rc = upload(aids.radii.data(), sizeof(double) * ne, drad, st))) return rc;
    if ((rc = upload(aids.tiles.data(), sizeof(double) * aids.tiles.size(), dtil, st))) return rc;
  } else {
    dist_wind_kernel<2><<<grid, kThreads, 0, st>>>(src, (const double*)de.p, ne, m, (double*)dxi.p, (double*)dwind.p);
  }
  GF_CUDA(cudaGetLastError());
  GF_CUDA(cudaEventRecord(ev[1], st));
  if (family != 0) {
    // xi_eff = max(xi, eta_min) (descriptor.py:338)
    GF_CUDA(dxe.alloc(sizeof(double) * m));
    clamp_min_kernel<<<sm_count() * 8, 256, 0, st>>>((const double*)dxi.p, (double*)dxe.p, m, eta_min);
    GF_CUDA(cudaGetLastError());
    SweepParams sp = {sigma, gconst, max_angle, eta_min, 1.0 / (2.5066282746310002 * sigma), max_depth,
                      max_angle * (1.0 - 1e-9)};
    const unsigned sgrid = (unsigned)ceil_div(m, kSweepThreads);
    if (d == 3)
      sweep_kernel<3><<<sgrid, kSweepThreads, 0, st>>>(src, (const double*)de.p, (const double*)dn.p,
                                                       (const double*)dm.p, (const double*)drad.p,
                                                       (const double*)dtil.p, ne, m, (const double*)dxe.p, sp,
                                                       (double*)dip.p, (double*)dres.p, (int64_t*)dcl.p);
    else
      sweep_kernel<2><<<sgrid, kSweepThreads, 0, st>>>(src, (const double*)de.p, (const double*)dn.p,
                                                       (const double*)dm.p, nullptr, nullptr, ne, m,
                                                       (const double*)dxe.p, sp, (double*)dip.p, (double*)dres.p,
                                                       (int64_t*)dcl.p);
    GF_CUDA(cudaGetLastError());
  }
  GF_CUDA(cudaEventRecord(ev[2], st));
  combine_kernel<<<sm_count() * 8, 256, 0, st>>>(m, (const double*)dxi.p, (const double*)dwind.p, (const double*)dip.p,
                                          (const double*)dres.p, family, lam_in, lam_out, eta_min, max_angle,
                                          (double*)dval.p, out_flags);
  GF_CUDA(cudaGetLastError());
  neighbor_fill_kernel<<<sm_count() * 8, 256, 0, st>>>(d, src.dims[0], src.dims[1], d == 3 ? src.dims[2] : 1,
                                                (const double*)dval.p, out_flags, (double*)out_vals);
  GF_CUDA(cudaGetLastError());
  if (halos) {
    GF_CUDA(cudaMemcpyAsync(values_dev, (const double*)out_vals + 2 * off, sizeof(double) * 2 * own,
                            cudaMemcpyDeviceToDevice, st));
    GF_CUDA(cudaMemcpyAsync(flags_dev, out_flags + off, own, cudaMemcpyDeviceToDevice, st));
  }
  DevBuf dst;
  GF_CUDA(dst.alloc(2 * sizeof(unsigned long long)));
  GF_CUDA(cudaMemsetAsync(dst.p, 0, 2 * sizeof(unsigned long long), st));
  stats_kernel<<<sm_count() * 4, 256, 0, st>>>((const double*)dres.p + off, (const int64_t*)dcl.p + off, own,
                                        (unsigned long long*)dst.p);
  GF_CUDA(cudaGetLastError());
  unsigned long long hs[2];
  GF_CUDA(cudaMemcpyAsync(hs, dst.p, sizeof hs, cudaMemcpyDeviceToHost, st));
  GF_CUDA(cudaStreamSynchronize(st));
  stats[0] = (double)hs[0];
  stats[1] = __longlong_as_double_host(hs[1]);
  float ms_dw = 0.f, ms_sw = 0.f;
  GF_CUDA(cudaEventElapsedTime(&ms_dw, ev[0], ev[1]));
  GF_CUDA(cudaEventElapsedTime(&ms_sw, ev[1], ev[2]));
  stats[2] = 1e-3 * ms_dw;
  stats[3] = 1e-3 * ms_sw;
  return 0;
}

int gf_affinity_grid(int d, const double* elems, const double* normals, const double* measures, int64_t ne,
                     const int32_t* dims, const double* origin, double spacing, int family, double sigma,
                     double gconst, double lam_in, double lam_out, double max_angle, int max_depth, double eta_floor,
                     void* values_dev, uint8_t* flags_dev, double* stats, void* stream) {
  GF_CHECK(dims != nullptr, GF_EINVAL, "bad argument");
  return gf_affinity_planes(d, elems, normals, measures, ne, dims, origin, spacing, 0, dims[0], 0, 0, family, sigma,
                            gconst, lam_in, lam_out, max_angle, max_depth, eta_floor, values_dev, flags_dev, stats,
                            stream);
}

}  // extern "C"
