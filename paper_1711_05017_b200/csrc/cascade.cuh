// cascade.cuh -- launch interface of the cascade (query / pose sweep) kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gf {

constexpr int kNumMoments = 26;  // S(2) + Z[3](6) + Y[3][3](18), see cascade.cu

struct CascadeArgs {
  const void* C1;        // raw window, complex<T>, (w0, w1, w2) row-major
  const void* C2p;       // packed moving window (see pack_window_kernel)
  int w[3];
  int dim;               // 2 or 3 (2D windows run as w2 = 1)
  int wrap;
  int precision;         // 32 or 64
  double dom[3];         // frequency spacing per axis
  double rdom[3][3];     // dom[i] / dom[j] (host-computed)
  double dcell;          // 1 / (N^d dV)
  double center[3];      // grid centre c
  // poses: `poses` (device, n x 12 doubles: R row-major then t_eff) or,
  // when null, the single pose carried in the launch parameters
  const double* poses;
  double pose_inline[12];
  int64_t pose_offset;
  // work decomposition (filled by plan_cascade)
  int seg_len;
  int segs_per_row;
  int64_t n_seg;
  int blocks_per_pose;
  int64_t segs_per_block;
  double tie_eps;
  int single;            // 1: one pose through the latency kernel (cascade_single.cu)
  int pdl;               // 1: launch with programmatic dependent launch (serial loop)
  // cross-block scratch and output
  double* partials;      // n_poses * blocks_per_pose * kNumMoments (if bpp > 1)
  unsigned* counters;    // n_poses, zero-initialised, re-armed by the kernel
  // serial loop scratch ring (null: one scratch set, guarded by griddepcontrol.wait):
  // this query's slot may be written once *slot_done >= slot_need (every
  // earlier user of the slot has read it back); the finishing CTA then
  // publishes slot_need + 1
  unsigned* slot_done;
  unsigned slot_need;
  double* out;           // n_poses * 14 (interleaved complex128 x 7)
  unsigned long long* debug;  // optional per-block phase timestamps (single kernel)
  // single kernel, host-polled result: 28 host-mapped 8-byte slots, slot 2i+h
  // = (seq32 << 32) | 32-bit half h of output i.  Each slot is one atomic
  // 8-byte store carrying its own validity tag, so the host needs no separate
  // completion word and the kernel no system-scope fence (or null: `out`).
  unsigned long long* ll_out;
  unsigned long long done_seq;  // tag of this query
  // resident server only: globaltimer when the lead CTA saw the request; the
  // finishing CTA reports (now - *t_detect) as a tagged 29th result slot
  unsigned long long* t_detect;
};

// 26 moment accumulators (layout = the moment index order used by finalize)
template <typename T> struct Acc26 {
  T v[kNumMoments];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < kNumMoments; ++i) v[i] = (T)0;
  }
  // S += bV; Z_a += k_a bV; Y[b][a] += k_a X_b
  template <typename C>
  __device__ __forceinline__ void add(C bV, C X0, C X1, C X2, T kx, T ky, T kz) {
    v[0] += bV.re; v[1] += bV.im;
    v[2] = fma(kx, bV.re, v[2]); v[3] = fma(kx, bV.im, v[3]);
    v[4] = fma(ky, bV.re, v[4]); v[5] = fma(ky, bV.im, v[5]);
    v[6] = fma(kz, bV.re, v[6]); v[7] = fma(kz, bV.im, v[7]);
    const C X[3] = {X0, X1, X2};
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      v[8 + 6 * b] = fma(kx, X[b].re, v[8 + 6 * b]);  v[9 + 6 * b] = fma(kx, X[b].im, v[9 + 6 * b]);
      v[10 + 6 * b] = fma(ky, X[b].re, v[10 + 6 * b]); v[11 + 6 * b] = fma(ky, X[b].im, v[11 + 6 * b]);
      v[12 + 6 * b] = fma(kz, X[b].re, v[12 + 6 * b]); v[13 + 6 * b] = fma(kz, X[b].im, v[13 + 6 * b]);
    }
  }
};

// Persistent haptic server mailbox plumbing (cascade_single.cu)
// Persistent server mailbox: kReqSlots 8-byte slots, (seq32 << 32) | payload:
// slots 0..23 the 32-bit halves of the pose (R row-major, then t_eff), slot
// 24 the stop word.  A request is complete when every slot carries its tag.
constexpr int kReqSlots = 25;
struct ServerCtl {
  const volatile unsigned long long* host_req;  // host-mapped request slots
  volatile unsigned long long* dev_req;         // device copy forwarded by CTA 0
  unsigned long long start_seq;
  unsigned long long idle_timeout_ns;
  int sm_limit;         // clusters whose rank 0 runs on an SM id >= sm_limit leave at start
  unsigned* enlist;     // 2 zeroed device counters: clusters decided, clusters serving
};
cudaError_t launch_cascade_server(const CascadeArgs& a, const ServerCtl& ctl, cudaStream_t st);

// Grid of the single-pose kernels (measured, profiles/r02_cascade_grid.txt):
// the lone query and the serial loop run one CTA per SM -- a programmatic
// dependent launch's CTAs then fit beside the previous query's (serial loop
// w = 64: 4.8 us/query against 6.7 at two per SM); the resident server, whose
// queries cannot overlap, runs two per SM (7.9 us against 9.1 at one).
constexpr int kLaunchCtasPerSm = 1;
constexpr int kServerCtasPerSm = 2;
int single_blocks(const CascadeArgs& a, int target_blocks);
cudaError_t launch_cascade_single(const CascadeArgs& a, cudaStream_t st);
void plan_cascade(CascadeArgs& a, int64_t n_poses, int target_blocks);
cudaError_t launch_cascade(const CascadeArgs& a, int64_t n_poses, cudaStream_t st);
int64_t packed_window_elems(const int w[3]);
cudaError_t launch_pack_window(int precision, const void* raw, void* packed, const int w[3], int wrap,
                               cudaStream_t st);
cudaError_t launch_narrow(const void* src, void* dst, int64_t n, cudaStream_t st);

}  // namespace gf
