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
  // cross-block scratch and output
  double* partials;      // n_poses * blocks_per_pose * kNumMoments (if bpp > 1)
  unsigned* counters;    // n_poses, zero-initialised, re-armed by the kernel
  double* out;           // n_poses * 14 (interleaved complex128 x 7)
};

void plan_cascade(CascadeArgs& a, int64_t n_poses, int target_blocks);
cudaError_t launch_cascade(const CascadeArgs& a, int64_t n_poses, cudaStream_t st);
int64_t packed_window_elems(const int w[3]);
cudaError_t launch_pack_window(int precision, const void* raw, void* packed, const int w[3], int wrap,
                               cudaStream_t st);
cudaError_t launch_narrow(const void* src, void* dst, int64_t n, cudaStream_t st);

}  // namespace gf
