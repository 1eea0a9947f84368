// cascade_single.cu -- latency kernel for ONE pose (the haptic query, Q1),
// one-shot or as a resident server.
//
// Same semantics as cascade.cu (reference _core.cascade_3d,
// /root/reference/pkg/src/geofield/_core.pyx:598-724).  A lone query has
// only ~10^5-10^6 modes, so latency is set by the setup, the per-thread
// dependency chain and the cross-CTA reduction tail, not by bandwidth:
//   * setup: per-axis translation-phase tables (sincospi of float64-reduced
//     arguments), 32.32 fixed-point index coefficients, the lane orientation
//     and -- for lattice-aligned poses -- the tie tables, all from the pose
//     in one pass and one barrier;
//   * mode loop: 148 CTAs of 256 threads for a launch (two per SM for the
//     resident server, cascade.cuh kLaunchCtasPerSm / kServerCtasPerSm);
//     the serial loop chains launches by programmatic dependent launch over
//     a 4-slot scratch ring (up to three queries in flight); each CTA walks a contiguous
//     run of units (consecutive run-axis planes of one oriented 4 x 8 lane
//     patch), so the fixed-point index advances by exact integer adds, the
//     p/q phase product is reused and consecutive gathers reuse L1 lines;
//   * reduction: 26 moments through a conflict-free shared-memory transpose,
//     cluster ranks push their block moments to the cluster leader through
//     DSMEM (mbarrier hand-off), leaders write partials, and the last leader
//     (integer ticket) sums them in fixed order -- bitwise repeatable;
//   * result: 28 self-tagged 8-byte words written to host-mapped memory, so
//     the host needs no completion flag and the kernel no system fence.
// The server variant keeps the grid resident (cooperative + clustered
// launch); CTA 0 polls the host mailbox and forwards each pose through L2.
#include "cascade.cuh"
#include "common.cuh"

#include <cooperative_groups.h>
#include <cuda/atomic>

#include <math.h>

namespace gf {
namespace {

constexpr int kThreads = 256;
// transpose row stride: = 8 (mod 32) so the reduction's reads -- lanes (c, s)
// at c * kTrLd + s + 8 i -- hit 32 distinct banks (fp32) / distinct 8-byte
// slots per half-warp (fp64)
constexpr int kTrLd = kThreads + 8;
constexpr int kCluster = 4;  // CTAs per cluster (DSMEM reduction stage; measured best, profiles/r01_summary.md)

struct SinglePose {
  double mu[3][3];
  double R[9];
  double targ[3];
  int p, q, r, nP, nQ;
  // this CTA's unit range [u_begin, u_end) as (run, plane) of its first unit
  // and the run as (p tile, q tile): one thread divides, the others read
  int u_begin, u_end, run0, kr00, rp0, rq0;
  // finalize coefficients (computed during setup, used by the last block):
  double cg[3][3][3];  // G_g += cg[g][b][a] * Y[b][a]  (= -A_g[a][b] dw_a / dw_b)
  double kq[3][3];     // G_g += 2 pi i kq[g][a] Z_a     (= dw_a q_g[a])
  double kt[3];        // T_a  = 2 pi i kt[a] Z_a        (= dw_a)
  long long ufix[3][4];  // fixed-point u_a = ufix[a][3] + sum_b ufix[a][b] kappa_b
  int tie_dep[3];  // column a of R has one nonzero, in row tie_dep[a] (else -1): see tie table
};

// Cluster stage state (shared memory of every CTA; used in rank 0): the
// other ranks push their 26 block moments into `gather` with DSMEM stores
// and arrive on `bar` (release.cluster); rank 0 waits on it (acquire) -- a
// one-way hand-off, no cluster-wide barrier on the query path.
constexpr int kMaxCluster = 8;
static_assert(kCluster <= kMaxCluster, "cluster stage sized for kMaxCluster ranks");
// resident CTAs per SM the register budget is sized for: the server grid is
// kServerCtasPerSm x 148 CTAs (up to 128 registers); the one-shot kernel runs
// kLaunchCtasPerSm per SM and keeps room for four (64 registers), so the CTAs
// of the next launches of a PDL chain start beside the previous tail
// (cascade.cuh; serial loop w = 64: 4.46 -> 4.31 us/query against room for
// three, the lone launch ~3 % slower -- profiles/r02_cascade_grid.txt)
constexpr int kMinBlocksServer = kServerCtasPerSm;
constexpr int kMinBlocksLaunch = 4;
struct ClusterRed {
  double gather[kMaxCluster][kNumMoments];
  unsigned long long bar;
  unsigned parity;  // phase of `bar` for the next query
  int armed;        // 1 until the start-of-kernel cluster barrier has been waited on
};

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned map_rank0(unsigned addr) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(addr));
  return r;
}

// Kernel start: rank 0 initialises the hand-off barrier; every CTA arrives
// (relaxed) on the cluster barrier and waits for it lazily before its first
// push, so the init is visible without a barrier on the critical path.
__device__ __forceinline__ void cluster_red_init(ClusterRed& cr) {
  unsigned crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  if (threadIdx.x == 0) {
    cr.parity = 0;
    cr.armed = 1;
    if (crank == 0 && csize > 1) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&cr.bar)), "r"(csize - 1));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  if (csize > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}

__device__ __forceinline__ double exact_u_s(const double* R, const double* dom, int a, int kx, int ky, int kz,
                                            int hx, int hy, int hz, int ha) {
  double ox = __dmul_rn((double)(kx - hx), dom[0]);
  double oy = __dmul_rn((double)(ky - hy), dom[1]);
  double oz = __dmul_rn((double)(kz - hz), dom[2]);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(R[0 + a], ox), __dmul_rn(R[3 + a], oy)), __dmul_rn(R[6 + a], oz));
  return __dadd_rn(__ddiv_rn(-s, dom[a]), (double)ha);
}

// A_g[ax][bb] = (Omega_g R)[ax][bb] for row-major R, Omega_g the generator
// of rotations about axis g: -eps(g, ax, c) R[c][bb] with c the third axis
// (0 when g == ax) -- selects, no lane-divergent branches in the setup
__device__ __forceinline__ double gen_rot(const double* R, int g, int ax, int bb) {
  const int c = 3 - g - ax;
  const double v = R[3 * ((unsigned)c > 2u ? 0 : c) + bb];
  return g == ax ? 0.0 : ((ax - g + 3) % 3 == 1 ? -v : v);
}

// tie-table floor stored in the real slot: as raw int bits for fp32 (no
// int<->float conversion in the mode loop), as a value for fp64
__device__ __forceinline__ float pack_floor(int v, float) { return __int_as_float(v); }
__device__ __forceinline__ double pack_floor(int v, double) { return (double)v; }
__device__ __forceinline__ int unpack_floor(float v) { return __float_as_int(v); }
__device__ __forceinline__ int unpack_floor(double v) { return (int)v; }

// Output slot i (0..13, interleaved complex) as a linear form of the 26
// moments, from the coefficients precomputed in setup (14 threads).
__device__ __forceinline__ double finalize_slot(const CascadeArgs& a, const SinglePose& sp, const double* m, int i) {
  const double TWO_PI = 6.283185307179586;
  const double dc = a.dcell;
  if (i < 2) return dc * m[i];
  if (i < 8) {  // T_a = 2 pi i dw_a Z_a
    const int ax = (i - 2) >> 1;
    const double k = dc * TWO_PI * sp.kt[ax];
    return (i & 1) ? k * m[2 + 2 * ax] : -k * m[3 + 2 * ax];
  }
  const int g = (i - 8) >> 1, im = i & 1;
  double acc = 0.0;
#pragma unroll
  for (int bb = 0; bb < 3; ++bb)
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) acc += sp.cg[g][bb][ax] * m[8 + im + 2 * (3 * bb + ax)];
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double k = TWO_PI * sp.kq[g][ax];
    acc += im ? k * m[2 + 2 * ax] : -k * m[3 + 2 * ax];
  }
  return dc * acc;
}

// Result of one query: slot i of 14 to `out`, or as two self-tagged 8-byte
// words to the host-mapped LL slots (plain stores, no fence: the host checks
// the tags).
__device__ __forceinline__ void emit_output(const CascadeArgs& a, int i, double v, unsigned long long seq) {
  if (a.ll_out) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned long long tag = (seq & 0xffffffffull) << 32;
    volatile unsigned long long* o = a.ll_out;
    o[2 * i] = tag | (bits & 0xffffffffull);
    o[2 * i + 1] = tag | (bits >> 32);
  } else {
    a.out[i] = v;
  }
}

// Resident server: the low words of the globaltimer at request detection and
// at the result, as tagged slots 28 and 29 -- per-frame diagnostics that
// tell a slow GPU answer from a host or PCIe stall (the host stamps its own
// post and receipt times beside them).
__device__ __forceinline__ void emit_timing(const CascadeArgs& a, unsigned long long seq) {
  if (!a.t_detect || !a.ll_out) return;
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  const unsigned long long det = *(volatile unsigned long long*)a.t_detect;
  const unsigned long long tag = (seq & 0xffffffffull) << 32;
  const unsigned long long gap = *(volatile unsigned long long*)(a.t_detect + 1);
  volatile unsigned long long* o = a.ll_out;
  o[28] = tag | (det & 0xffffffffull);
  o[29] = tag | (now & 0xffffffffull);
  o[30] = tag | (gap > 0xffffffffull ? 0xffffffffull : gap);
  const unsigned long long cgap = *(volatile unsigned long long*)(a.t_detect + 2);
  o[31] = tag | (cgap > 0xffffffffull ? 0xffffffffull : cgap);
}

// Serial-loop scratch ring (CascadeArgs::slot_done): wait until every earlier
// user of this query's slot has published its release (one poller, then the
// CTA barrier orders the slot writes after its acquire).
__device__ __forceinline__ void ring_slot_acquire(const CascadeArgs& a, int tid) {
  if (tid == 32) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.slot_done) : "memory");
      if (v >= a.slot_need) break;
      __nanosleep(32);
    }
  }
  __syncthreads();
}

// ring mode: a query's grid completes only after its predecessor's, so work
// stream-ordered after the chain sees every query finished
__device__ __forceinline__ void ring_exit(bool ring) {
  if (ring) asm volatile("griddepcontrol.wait;" ::: "memory");
}

// One pose over all retained modes, spread across the grid; shared state is
// passed in so the same body runs in the one-shot kernel and in the
// persistent haptic server.  Non-final blocks return early (block-uniform).
template <typename T, bool WRAP>
__device__ __forceinline__ void single_pose_body(const CascadeArgs& a, const double* src, SinglePose& sp, double* red,
                                                 unsigned& ticket, ClusterRed& cr, unsigned char* smem_raw,
                                                 unsigned long long done_seq, int vb, int vg) {
  using P4 = typename pair4<T>::type;
  // dynamic: transpose buffer tr[26][257] (reduction) | px | py | pz
  T(*tr)[kTrLd] = reinterpret_cast<T(*)[kTrLd]>(smem_raw);
  cx<T>* ptab = reinterpret_cast<cx<T>*>(smem_raw + sizeof(T) * kNumMoments * kTrLd + 16);
  // tie table: for an axis a whose R column has a single nonzero (row b --
  // lattice-aligned poses: identity, screws about a grid axis) the reference
  // index u_a depends on k_b alone, and on such poses EVERY mode sits on an
  // integer u_a.  Its float64 reference floor and fraction are tabulated
  // once per pose at [offset(b) + k_b] (distinct b per a: R is a rotation)
  // as (floor, frac) in T, so the tie branch is one shared load instead of a
  // float64 divide and three float64 conversions per mode.
  cx<T>* ttab = ptab + (a.w[0] + a.w[1] + a.w[2]);

  const int tid = threadIdx.x;
  unsigned long long* dbg = a.debug ? a.debug + (int64_t)vb * 8 : nullptr;
#define GF_STAMP(k)                                                                 \
  if (dbg && tid == 0) {                                                           \
    unsigned long long t_;                                                         \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                         \
    dbg[k] = t_;                                                                   \
  }
  GF_STAMP(0)
  const int w0 = a.w[0], w1 = a.w[1], w2 = a.w[2];
  const int hx = w0 / 2, hy = w1 / 2, hz = w2 / 2;
  if (tid < 9) {
    sp.R[tid] = src[tid];
    int ia = tid / 3, ib = tid % 3;
    sp.mu[ia][ib] = -src[ib * 3 + ia] * a.rdom[ib][ia];
  }
  if (tid >= 32 && tid < 32 + 27) {  // A_g = Omega_g R (_core.pyx:615-626)
    const int k = tid - 32, g = k / 9, bb = (k / 3) % 3, ax = k % 3;
    sp.cg[g][bb][ax] = -gen_rot(src, g, ax, bb) * a.rdom[ax][bb];
  }
  if (tid >= 64 && tid < 64 + 9) {  // q_g = A_g c
    const int g = (tid - 64) / 3, ax = (tid - 64) % 3;
    double q = 0.0;
#pragma unroll
    for (int bb = 0; bb < 3; ++bb) q += gen_rot(src, g, ax, bb) * a.center[bb];
    sp.kq[g][ax] = a.dom[ax] * q;
  }
  if (tid >= 96 && tid < 99) sp.kt[tid - 96] = a.dom[tid - 96];
  if (tid >= 128 && tid < 140) {
    const int ia = (tid - 128) / 4, ib = (tid - 128) % 4;
    sp.ufix[ia][ib] = ib == 3 ? to_fix32((double)(ia == 0 ? hx : (ia == 1 ? hy : hz)))
                              : to_fix32(-src[ib * 3 + ia] * a.rdom[ib][ia]);
  }
  if (tid == 160) {  // lane order for this pose (warp 5, from the pose itself: no barrier before it)
    const double z0 = fabs(src[2] * a.rdom[0][2]), z1 = fabs(src[5] * a.rdom[1][2]),
                 z2 = fabs(src[8] * a.rdom[2][2]);  // |mu[2][b]|
    int r = 2;
    if (a.dim == 3) r = z0 <= z1 ? 0 : 1;  // never z: C1 loads along z runs scatter (cascade.cu)
    int o1 = (r + 1) % 3, o2 = (r + 2) % 3;
    if (a.dim == 2) { o1 = 0; o2 = 1; }
    const double zo1 = o1 == 0 ? z0 : (o1 == 1 ? z1 : z2), zo2 = o2 == 0 ? z0 : (o2 == 1 ? z1 : z2);
    bool sw = zo1 > zo2;
    sp.p = sw ? o2 : o1;
    sp.q = sw ? o1 : o2;
    sp.r = r;
    sp.nP = ((sp.p == 0 ? w0 : (sp.p == 1 ? w1 : w2)) + 15) / 16;
    sp.nQ = ((sp.q == 0 ? w0 : (sp.q == 1 ? w1 : w2)) + 15) / 16;
    const int wr_ = r == 0 ? w0 : (r == 1 ? w1 : w2);
    const int units_ = sp.nP * sp.nQ * wr_;
    const int upb = (units_ + vg - 1) / vg;
    sp.u_begin = min(units_, vb * upb);
    sp.u_end = min(units_, sp.u_begin + upb);
    sp.run0 = sp.u_begin / wr_;
    sp.kr00 = sp.u_begin - sp.run0 * wr_;
    sp.rp0 = sp.run0 / sp.nQ;
    sp.rq0 = sp.run0 - sp.rp0 * sp.nQ;
  }
  if (tid == 192) {
    for (int ax = 0; ax < 3; ++ax) {
      const int nz = (src[ax] != 0.0) + (src[3 + ax] != 0.0) + (src[6 + ax] != 0.0);
      sp.tie_dep[ax] = nz != 1 ? -1 : (src[ax] != 0.0 ? 0 : (src[3 + ax] != 0.0 ? 1 : 2));
    }
  }
  // per-axis translation phase tables (and tie tables), concurrently with the sections above
  for (int i = tid; i < w0 + w1 + w2; i += kThreads) {
    int ax = i < w0 ? 0 : (i < w0 + w1 ? 1 : 2);
    int k = i - (ax == 0 ? 0 : (ax == 1 ? w0 : w0 + w1));
    int hh = ax == 0 ? hx : (ax == 1 ? hy : hz);
    // tie table entry: the axis c whose R column has its single nonzero in row ax
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const bool only = src[3 * ax + c] != 0.0 && src[3 * ((ax + 1) % 3) + c] == 0.0 && src[3 * ((ax + 2) % 3) + c] == 0.0;
      if (only) {
        const double ue = exact_u_s(src, a.dom, c, ax == 0 ? k : hx, ax == 1 ? k : hy, ax == 2 ? k : hz, hx, hy, hz,
                                    c == 0 ? hx : (c == 1 ? hy : hz));
        const double fe = floor(ue);
        ttab[i] = mk<T>(pack_floor((int)fe, T(0)), (T)(ue - fe));
      }
    }
    double cyc = (a.dom[ax] * src[9 + ax]) * (double)(k - hh);
    cyc -= rint(cyc);
    T sn, cs;
    if constexpr (sizeof(T) == 4) sincospif(2.0f * (float)cyc, &sn, &cs);
    else sincospi(2.0 * cyc, &sn, &cs);
    ptab[i] = mk<T>(cs, sn);
  }
  __syncthreads();

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

  Acc26<T> acc;
  acc.zero();
  GF_STAMP(1)
  // Each CTA takes a contiguous range of units; consecutive units are
  // consecutive run-axis planes of one (p, q) patch, so the range splits into
  // segments walked by the inner loop: the fixed-point index advances by one
  // exact integer add per axis, C1 by one stride, and the seven per-mode
  // products go into 8 run sums (sum Y, sum j Y) folded into the 26 moments
  // once per segment -- the batched sweep's loop shape (cascade.cu).
  const int u_begin = sp.u_begin, u_end = sp.u_end;
  const cx<T>* pt_p = ptab + (p == 0 ? 0 : (p == 1 ? w0 : w0 + w1));
  const cx<T>* pt_q = ptab + (q == 0 ? 0 : (q == 1 ? w0 : w0 + w1));
  const cx<T>* pt_r = ptab + (r == 0 ? 0 : (r == 1 ? w0 : w0 + w1));
  long long fxr = 0, fyr = 0, fzr = 0;  // d(u_a)/d(k_r) in 32.32 fixed point
  if constexpr (sizeof(T) == 4) {
    fxr = r == 0 ? sp.ufix[0][0] : (r == 1 ? sp.ufix[0][1] : sp.ufix[0][2]);
    fyr = r == 0 ? sp.ufix[1][0] : (r == 1 ? sp.ufix[1][1] : sp.ufix[1][2]);
    fzr = r == 0 ? sp.ufix[2][0] : (r == 1 ? sp.ufix[2][1] : sp.ufix[2][2]);
  }
  const T mr0 = r == 0 ? m00 : (r == 1 ? m01 : m02);  // fp64 engine: du_a / dk_r
  const T mr1 = r == 0 ? m10 : (r == 1 ? m11 : m12);
  const T mr2 = r == 0 ? m20 : (r == 1 ? m21 : m22);
  // axes read from the tie table (uniform over the block)
  const int tmask = (sp.tie_dep[0] >= 0 ? 1 : 0) | (sp.tie_dep[1] >= 0 ? 2 : 0) | (a.dim == 3 && sp.tie_dep[2] >= 0 ? 4 : 0);
  const int sr = r == 0 ? w1 * w2 : (r == 1 ? w2 : 1);  // C1 stride along the run axis
  const T er0 = r == 0 ? (T)1 : (T)0, er1 = r == 1 ? (T)1 : (T)0, er2 = r == 2 ? (T)1 : (T)0;
  // segment walk: (run, first plane) advance without divisions
  int rp = sp.rp0, rq = sp.rq0, kr_first = sp.kr00;
  for (int seg = u_begin; seg < u_end;) {
    const int kr0 = kr_first;
    const int kend = min(wr, kr0 + (u_end - seg));
    seg += kend - kr0;
    const int kp = 16 * rp + dp, kq = 16 * rq + dq;
    kr_first = 0;  // the next segment starts a new run
    if (++rq == sp.nQ) {
      rq = 0;
      ++rp;
    }
    if (kp >= wp || kq >= wq) continue;
    const int kx0 = p == 0 ? kp : (q == 0 ? kq : kr0);
    const int ky0 = p == 1 ? kp : (q == 1 ? kq : kr0);
    const int kz0 = p == 2 ? kp : (q == 2 ? kq : kr0);
    const T k0x = (T)(kx0 - hx), k0y = (T)(ky0 - hy), k0z = (T)(kz0 - hz);
    const cx<T> ph_pq = pt_p[kp] * pt_q[kq];
    long long fu3[3] = {0, 0, 0};
    T u0[3] = {(T)0, (T)0, (T)0};
    if constexpr (sizeof(T) == 4) {
      const int kk[3] = {kx0 - hx, ky0 - hy, kz0 - hz};
#pragma unroll
      for (int ax = 0; ax < 3; ++ax)
        fu3[ax] = sp.ufix[ax][3] + (long long)kk[0] * sp.ufix[ax][0] + (long long)kk[1] * sp.ufix[ax][1] +
                  (long long)kk[2] * sp.ufix[ax][2];
    } else {
      u0[0] = fma(m02, k0z, fma(m01, k0y, fma(m00, k0x, (T)hx)));
      u0[1] = fma(m12, k0z, fma(m11, k0y, fma(m10, k0x, (T)hy)));
      u0[2] = fma(m22, k0z, fma(m21, k0y, fma(m20, k0x, (T)hz)));
    }
    cx<T> rS = mk<T>(0, 0), rJ = mk<T>(0, 0);
    cx<T> rX[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
    cx<T> rXJ[3] = {mk<T>(0, 0), mk<T>(0, 0), mk<T>(0, 0)};
    int c1off = (kx0 * w1 + ky0) * w2 + kz0;
#pragma unroll(sizeof(T) == 4 ? 2 : 1)
    for (int kr = kr0; kr < kend; ++kr, c1off += sr) {
      const T j = (T)(kr - kr0);
      int il[3];
      T f[3];
      if constexpr (sizeof(T) == 4) {
        // exact 32.32 fixed-point index; float64 reference order only within 1e-6 of an integer
        unsigned lo[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          lo[ax] = fix_lo(fu3[ax]);
          il[ax] = fix_floor(fu3[ax]);
          f[ax] = fix_frac(lo[ax]);
        }
        fu3[0] += fxr;
        fu3[1] += fyr;
        fu3[2] += fzr;
        if (tmask) {  // lattice-aligned axes: the tabulated reference floor / frac, never a tie
          const int kx = r == 0 ? kr : kx0, ky = r == 1 ? kr : ky0, kz = r == 2 ? kr : kz0;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax)
            if ((tmask >> ax) & 1) {
              const int dep = sp.tie_dep[ax];
              const cx<T> e = ttab[dep == 0 ? kx : (dep == 1 ? w0 + ky : w0 + w1 + kz)];
              il[ax] = unpack_floor(e.re);
              f[ax] = e.im;
              lo[ax] = 0x80000000u;
            }
        }
        const bool tz = a.dim == 3 && fix_tie(lo[2]);
        if (fix_tie(lo[0]) || fix_tie(lo[1]) || tz) {
          const int kx = r == 0 ? kr : kx0, ky = r == 1 ? kr : ky0, kz = r == 2 ? kr : kz0;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            if ((ax < 2 || tz) && fix_tie(lo[ax])) {
              double ue = exact_u_s(sp.R, a.dom, ax, kx, ky, kz, hx, hy, hz, ax == 0 ? hx : (ax == 1 ? hy : hz));
              double fe = floor(ue);
              il[ax] = (int)fe;
              f[ax] = (T)(ue - fe);
            }
          }
        }
      } else {
        const T u[3] = {fma(j, mr0, u0[0]), fma(j, mr1, u0[1]), fma(j, mr2, u0[2])};
        bool tie[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
          const T fl = floor(u[ax]);
          il[ax] = (int)fl;
          f[ax] = u[ax] - fl;
          tie[ax] = !((tmask >> ax) & 1) && (ax < 2 || a.dim == 3) && (f[ax] < eps || f[ax] > (T)1 - eps);
        }
        if (tmask || tie[0] || tie[1] || tie[2]) {
          const int kx = r == 0 ? kr : kx0, ky = r == 1 ? kr : ky0, kz = r == 2 ? kr : kz0;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            if ((tmask >> ax) & 1) {
              const int dep = sp.tie_dep[ax];
              const cx<T> e = ttab[dep == 0 ? kx : (dep == 1 ? w0 + ky : w0 + w1 + kz)];
              il[ax] = unpack_floor(e.re);
              f[ax] = e.im;
            } else if (tie[ax]) {
              double ue = exact_u_s(sp.R, a.dom, ax, kx, ky, kz, hx, hy, hz, ax == 0 ? hx : (ax == 1 ? hy : hz));
              double fe = floor(ue);
              il[ax] = (int)fe;
              f[ax] = (T)(ue - fe);
            }
          }
        }
      }
      int ix = il[0], iy = il[1], iz = il[2];
      bool inside = true;
      if (WRAP) {
        ix = ix < 0 ? ix + w0 : (ix >= w0 ? ix - w0 : ix);
        iy = iy < 0 ? iy + w1 : (iy >= w1 ? iy - w1 : iy);
        iz = iz < 0 ? iz + w2 : (iz >= w2 ? iz - w2 : iz);
      } else if ((unsigned)(ix + 1) > (unsigned)w0 || (unsigned)(iy + 1) > (unsigned)w1 ||
                 (unsigned)(iz + 1) > (unsigned)w2) {
        // whole footprint outside the window: an exact zero contribution.
        // Predicated rather than skipped (base = 0 below, loads from a valid
        // cell), so the unrolled loop can issue the next modes' loads early.
        inside = false;
        ix = iy = iz = -1;
      }
      const P4* ptr = C2 + ((ix + 1) * sx + (iy + 1) * sy + (iz + 1));
      P4 e00 = ldg_pair(ptr), e10 = ldg_pair(ptr + sx), e01 = ldg_pair(ptr + sy), e11 = ldg_pair(ptr + sx + sy);
      const cx<T> base = inside ? C1[c1off] * (ph_pq * pt_r[kr]) : mk<T>(0, 0);
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
      if constexpr (sizeof(T) == 4) {
        rS += bV;
        axpy(rJ, j, bV);
        rX[0] += X0; rX[1] += X1; rX[2] += X2;
        axpy(rXJ[0], j, X0); axpy(rXJ[1], j, X1); axpy(rXJ[2], j, X2);
      } else {  // fp64 engine: straight into the moments (the run sums would spill)
        acc.add(bV, X0, X1, X2, fma(j, er0, k0x), fma(j, er1, k0y), fma(j, er2, k0z));
      }
    }
    if constexpr (sizeof(T) == 8) continue;
    // fold the segment: sum_j kappa_a(j) Y = kappa0_a sum Y + e_r,a sum j Y
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

  GF_STAMP(2)
  // ---- block reduction through a shared-memory transpose (fixed order)
#pragma unroll
  for (int c = 0; c < kNumMoments; ++c) tr[c][tid] = acc.v[c];
  __syncthreads();
  // 26 moments x 8 interleaved strands of 32 values: thread (c, s) sums
  // tr[c][s + 8 i], i < 32 (conflict-free, see kTrLd), fixed order
  double part = 0.0;
  const int c = tid >> 3, s = tid & 7;
  if (c < kNumMoments) {
    T q0 = (T)0, q1 = (T)0, q2 = (T)0, q3 = (T)0;  // 4 independent chains
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      q0 += tr[c][s + 8 * i];
      q1 += tr[c][s + 8 * (i + 1)];
      q2 += tr[c][s + 8 * (i + 2)];
      q3 += tr[c][s + 8 * (i + 3)];
    }
    part = (double)((q0 + q1) + (q2 + q3));
  }
  // combine the 8 segments of each moment (lanes 8 apart inside one warp)
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o, 8);
  if (c < kNumMoments && s == 0) red[c] = part;
  __syncthreads();

  // Programmatic dependent launch (the serial loop).  One scratch set: the
  // partials and ticket below are shared with the previous query, so wait for
  // its grid to complete here (everything above -- pose setup, mode loop --
  // overlapped its tail; a no-op without a PDL launch).  Scratch ring
  // (a.slot_done): the previous queries use other slots, so only this slot's
  // last user is awaited, at the partials store; the grid-completion wait
  // moves to the exit (ring_exit), which keeps the stream order of the chain.
  const bool ring = a.slot_done != nullptr;
  const int bpp = vg;
  if (bpp == 1) {
    if (tid < 14) emit_output(a, tid, finalize_slot(a, sp, red, tid), done_seq);
    if (tid == 14) emit_timing(a, done_seq);
    ring_exit(ring);
    return;
  }
  GF_STAMP(3)
  if (!ring) asm volatile("griddepcontrol.wait;" ::: "memory");
  // ---- cluster stage: ranks 1.. push their block moments to rank 0 through
  // distributed shared memory; rank 0 sums them in rank order (fixed)
  unsigned crank, csize;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  // (csize is kCluster, or 1 when the launch fell back to no clusters)
  const int cid = csize == kCluster ? vb / kCluster : vb, nclusters = csize == kCluster ? vg / kCluster : vg;
  if (csize > 1) {
    if (cr.armed) {  // rank 0's barrier init is visible once the start barrier completes
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      if (tid == 0) cr.armed = 0;
    }
    if (crank != 0) {
      if (tid < kNumMoments)
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(map_rank0(smem_addr(&cr.gather[crank][tid]))),
                     "d"(red[tid])
                     : "memory");
      __syncthreads();
      if (tid == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(map_rank0(smem_addr(&cr.bar)))
                     : "memory");
      ring_exit(ring);
      return;
    }
    double v = 0.0;
    if (tid < kNumMoments) {
      const unsigned bar = smem_addr(&cr.bar), par = cr.parity;
      unsigned done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(bar), "r"(par)
            : "memory");
      v = red[tid];
      for (unsigned r = 1; r < csize; ++r) v += cr.gather[r][tid];
    }
    if (ring) ring_slot_acquire(a, tid);  // ends with __syncthreads
    if (tid < kNumMoments) a.partials[(int64_t)tid * nclusters + cid] = v;  // moment-major
    __syncthreads();
    if (tid == 0) cr.parity ^= 1u;
  } else {
    if (ring) ring_slot_acquire(a, tid);
    if (tid < kNumMoments) a.partials[(int64_t)tid * nclusters + cid] = red[tid];
  }
  // ---- grid stage: integer ticket with release/acquire ordering
  __syncthreads();
  if (tid == 0) {
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> ctr(*a.counters);
    ticket = ctr.fetch_add(1u, cuda::memory_order_acq_rel);
  }
  __syncthreads();
  GF_STAMP(4)
  if (ticket != (unsigned)(nclusters - 1)) {
    ring_exit(ring);
    return;
  }
  // last leader: 26 moments x 8 segments, independent loads, fixed order
  double part2 = 0.0;
  if (c < kNumMoments) {
    const double* row = a.partials + (int64_t)c * nclusters;
    double q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = s + 8 * i;
      q[i] = b < nclusters ? __ldcg(row + b) : 0.0;
    }
    part2 = ((q[0] + q[1]) + (q[2] + q[3])) + ((q[4] + q[5]) + (q[6] + q[7]));
    for (int b = s + 64; b < nclusters; b += 8) part2 += __ldcg(row + b);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) part2 += __shfl_down_sync(0xffffffffu, part2, o, 8);
  if (c < kNumMoments && s == 0) red[c] = part2;
  __syncthreads();
  if (tid < 14) emit_output(a, tid, finalize_slot(a, sp, red, tid), done_seq);
  if (tid == 14) emit_timing(a, done_seq);
  if (tid == 0) {
    a.counters[0] = 0u;
    if (ring)  // the slot's partials are read (the barrier above) and its ticket re-armed
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.slot_done), "r"(a.slot_need + 1u) : "memory");
  }
  GF_STAMP(5)
  ring_exit(ring);
}

template <typename T, bool WRAP>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? kMinBlocksLaunch : 2) cascade3d_single_kernel(CascadeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SinglePose sp;
  __shared__ double red[kNumMoments];
  __shared__ unsigned ticket;
  __shared__ ClusterRed cr;
  __shared__ double pose_s[12];
  // pose to shared memory with direct (constant-bank) parameter reads: a
  // generic pointer into the parameter block turns every use into a global
  // load of freshly written launch memory on the setup critical path
  if (threadIdx.x < 12)
    pose_s[threadIdx.x] = a.poses ? a.poses[a.pose_offset * 12 + threadIdx.x] : a.pose_inline[threadIdx.x];
  // let the next query of a PDL launch sequence start its setup now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  cluster_red_init(cr);  // ends with __syncthreads
  single_pose_body<T, WRAP>(a, pose_s, sp, red, ticket, cr, smem_raw, a.done_seq, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// Persistent haptic server: the grid stays resident (cooperative launch) and
// serves one query per mailbox sequence number.  The lead CTA polls the host-
// mapped mailbox and forwards the pose to device memory; the other CTAs poll
// that device copy.  No kernel launch per query.
//
// SM budget (landscape exports run while a session serves
// frames): the grid is launched on every SM, then each cluster whose rank-0
// CTA sits on an SM id >= ctl.sm_limit exits at once, so those SMs stay free
// for other kernels for the whole session.  Survivors take dense virtual
// cluster ids from a device counter and split the modes among themselves.
constexpr unsigned long long kServerStop = ~0ull;
constexpr int kPollWarps = 2;  // lead-CTA warps polling the host mailbox

// one-time start-up: decide survival per cluster and hand out virtual ids.
// Returns false when this CTA's cluster leaves the server.
__device__ __forceinline__ bool server_enlist(const ServerCtl& ctl, int& vb, int& vg) {
  __shared__ int s_vcid, s_nsurv;
  unsigned crank, csize, smid;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const unsigned nclusters = gridDim.x / csize;
  if (threadIdx.x == 0) s_vcid = -1;
  __syncthreads();
  if (crank == 0 && threadIdx.x == 0) {
    // cluster 0 always serves, so at least one cluster survives any budget
    const bool keep = (blockIdx.x == 0) || smid < (unsigned)ctl.sm_limit;
    if (keep) s_vcid = (int)atomicAdd(ctl.enlist + 1, 1u);
    __threadfence();
    atomicAdd(ctl.enlist, 1u);
    // every cluster has decided once the first counter reaches the launch count
    while (*(volatile unsigned*)ctl.enlist < nclusters) __nanosleep(100);
    __threadfence();
    s_nsurv = (int)*(volatile unsigned*)(ctl.enlist + 1);
  }
  // rank 0's decision to the other ranks of the cluster (DSMEM read)
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  int vcid, nsurv;
  {
    unsigned a0 = map_rank0(smem_addr(&s_vcid)), a1 = map_rank0(smem_addr(&s_nsurv));
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(vcid) : "r"(a0) : "memory");
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(nsurv) : "r"(a1) : "memory");
  }
  // rank 0 must not exit while peers still read its shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (vcid < 0) return false;
  vb = vcid * (int)csize + (int)crank;
  vg = nsurv * (int)csize;
  return true;
}

template <typename T, bool WRAP>
__global__ void __launch_bounds__(kThreads, kMinBlocksServer) cascade3d_server_kernel(CascadeArgs a,
                                                                                               ServerCtl ctl) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SinglePose sp;
  __shared__ double red[kNumMoments];
  __shared__ unsigned ticket;
  __shared__ unsigned long long cur;
  __shared__ double pose_s[12];
  __shared__ ClusterRed cr;
  int vb = 0, vg = 1;
  if (!server_enlist(ctl, vb, vg)) return;  // this SM stays free for other work
  cluster_red_init(cr);
  unsigned long long last = ctl.start_seq;
  const int tid = threadIdx.x;
  const bool lead = vb == 0;
  __shared__ int found;  // lead CTA: which warp owns this request (0 = none yet)
  while (true) {
    const unsigned expect = (unsigned)(last + 1);
    if (tid == 0) found = 0;
    __syncthreads();
    // the lead CTA polls the host mailbox with kPollWarps warps whose polls
    // are staggered in time: a PCIe read takes ~1 us, so several reads in
    // flight cut the wait between the host's write and its detection.  The
    // first warp to see a complete request (or, warp 0 only, the idle
    // deadline) claims it with a CAS on `found`; only the owner forwards it.
    const int pollers = lead ? kPollWarps : 1;
    if (tid < 32 * pollers) {
      const int lane = tid & 31;
      unsigned long long v = 0;
      bool mine = true;
      if (lead) {
        const int pw = tid >> 5;
        unsigned long long t0, t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        do {  // stagger the start of warp pw by pw / kPollWarps of a PCIe round trip
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        } while (t1 - t0 < (unsigned long long)(pw * 1000 / kPollWarps));
        mine = false;
        unsigned long long t_prev = t1, gap = 0;  // longest stretch between two polls (diagnostics)
        while (true) {
          // .cv: treat any cached copy of the system-memory line as stale and fetch again
          if (lane < kReqSlots)
            asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(v) : "l"(ctl.host_req + lane) : "memory");
          bool got = __all_sync(0xffffffffu, lane >= kReqSlots || (unsigned)(v >> 32) == expect);
          bool stop_now = false;
          if (pw == 0) {  // only warp 0 may give up on idleness
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            gap = t1 - t_prev > gap ? t1 - t_prev : gap;
            t_prev = t1;
            stop_now = !got && t1 - t0 > ctl.idle_timeout_ns;
            if (got && lane == 0) *(volatile unsigned long long*)(a.t_detect + 1) = gap;
          }
          if (got || stop_now) {
            int won = 0;
            if (lane == 0) won = atomicCAS(&found, 0, pw + 1) == 0;
            won = __shfl_sync(0xffffffffu, won, 0);
            if (won) {
              mine = true;
              if (!got)  // idle: forward a stop request under this sequence number
                v = lane == kReqSlots - 1 ? (((unsigned long long)expect << 32) | 1ull)
                                          : ((unsigned long long)expect << 32);
            }
            break;
          }
          const int other = __shfl_sync(0xffffffffu, lane == 0 ? *(volatile int*)&found : 0, 0);
          if (other) break;  // another warp owns the request (warp-uniform)
        }
        if (mine && lane < kReqSlots) ctl.dev_req[lane] = v;
      } else {
        while (true) {
          if (lane < kReqSlots) v = ctl.dev_req[lane];
          const bool ok = __all_sync(0xffffffffu, lane >= kReqSlots || (unsigned)(v >> 32) == expect);
          if (ok) break;
          __nanosleep(20);
        }
      }
      // halves -> pose doubles (lanes 2i, 2i+1 -> pose_s[i]); stop word
      const unsigned lo = __shfl_sync(0xffffffffu, (unsigned)v, (2 * lane) & 31);
      const unsigned hi = __shfl_sync(0xffffffffu, (unsigned)v, (2 * lane + 1) & 31);
      const unsigned stopw = __shfl_sync(0xffffffffu, (unsigned)v, kReqSlots - 1);
      if (mine) {
        if (lane < 12) pose_s[lane] = __hiloint2double((int)hi, (int)lo);
        if (lane == 0) cur = stopw ? kServerStop : last + 1;
      }
    } else if (lead && tid >= 32 * kPollWarps && tid < 32 * (kPollWarps + 1)) {
      // diagnostics: a warp that only reads the clock while the pollers wait --
      // a long stretch here too means the SM stalled, not the PCIe read
      unsigned long long tp, tn, gap = 0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp));
      while (!*(volatile int*)&found) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tn));
        gap = tn - tp > gap ? tn - tp : gap;
        tp = tn;
      }
      if ((tid & 31) == 0) *(volatile unsigned long long*)(a.t_detect + 2) = gap;
    }
    __syncthreads();
    const unsigned long long sq = cur;
    if (sq == kServerStop) break;
    if ((a.debug || lead) && tid == 0) {  // when this CTA saw the query
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      if (a.debug) a.debug[(int64_t)vb * 8 + 7] = t_;
      if (lead) *(volatile unsigned long long*)a.t_detect = t_;
    }
    single_pose_body<T, WRAP>(a, pose_s, sp, red, ticket, cr, smem_raw, sq, vb, vg);
    last = sq;
    __syncthreads();
  }
  // a cluster's CTAs must not exit while a peer may still push into rank 0
  // (complete the start-up phase first if no query ever waited on it)
  if (cr.armed) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <typename T, bool WRAP>
cudaError_t launch_single_t(const CascadeArgs& a, cudaStream_t st) {
  size_t smem = sizeof(T) * kNumMoments * kTrLd + 16 + 2 * sizeof(cx<T>) * (a.w[0] + a.w[1] + a.w[2]);
  cudaError_t e = ensure_smem((const void*)cascade3d_single_kernel<T, WRAP>, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.blocks_per_pose);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // serial loop: programmatic dependent launch (see griddepcontrol in the body)
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, cascade3d_single_kernel<T, WRAP>, a);
}

}  // namespace

int single_blocks(const CascadeArgs& a, int target_blocks) {
  // units = nP * nQ * w_r, bounded by the orientation-independent worst case
  int64_t best = 0;
  for (int r = 0; r < 3; ++r) {
    int o1 = (r + 1) % 3, o2 = (r + 2) % 3;
    int64_t u = ceil_div(a.w[o1], 16) * ceil_div(a.w[o2], 16) * a.w[r];
    if (best == 0 || u < best) best = u;
  }
  const int64_t target = target_blocks;
  // equal work per CTA: the largest count <= target that gives every CTA the
  // same number of units (no straggler CTA with one extra unit)
  int64_t b = best < target ? best : target;
  if (best > target) b = best / ceil_div(best, target);
  b = (b / kCluster) * kCluster;  // whole clusters
  return (int)(b < kCluster ? kCluster : b);
}

template <typename T, bool WRAP>
cudaError_t launch_server_t(const CascadeArgs& a, const ServerCtl& ctl, cudaStream_t st) {
  size_t smem = sizeof(T) * kNumMoments * kTrLd + 16 + 2 * sizeof(cx<T>) * (a.w[0] + a.w[1] + a.w[2]);
  const void* fn = (const void*)cascade3d_server_kernel<T, WRAP>;
  cudaError_t e = ensure_smem(fn, smem);
  if (e != cudaSuccess) return e;
  const int per_sm = resident_ctas(fn, kThreads, smem);
  if ((int64_t)per_sm * sm_count() < a.blocks_per_pose) return cudaErrorCooperativeLaunchTooLarge;
  // co-residency guaranteed (cooperative) and the same CTA clusters as the
  // one-shot kernel (DSMEM hand-off stage)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.blocks_per_pose);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kCluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  e = cudaLaunchKernelEx(&cfg, cascade3d_server_kernel<T, WRAP>, a, ctl);
  if (e == cudaSuccess) return e;
  // clusters + cooperative refused (large fp64 windows): one-CTA clusters,
  // i.e. a plain cooperative launch -- the same body with csize = 1
  (void)cudaGetLastError();
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, cascade3d_server_kernel<T, WRAP>, a, ctl);
}

cudaError_t launch_cascade_server(const CascadeArgs& a, const ServerCtl& ctl, cudaStream_t st) {
  if (a.precision == 32)
    return a.wrap ? launch_server_t<float, true>(a, ctl, st) : launch_server_t<float, false>(a, ctl, st);
  return a.wrap ? launch_server_t<double, true>(a, ctl, st) : launch_server_t<double, false>(a, ctl, st);
}

cudaError_t launch_cascade_single(const CascadeArgs& a, cudaStream_t st) {
  if (a.precision == 32) return a.wrap ? launch_single_t<float, true>(a, st) : launch_single_t<float, false>(a, st);
  return a.wrap ? launch_single_t<double, true>(a, st) : launch_single_t<double, false>(a, st);
}

}  // namespace gf
