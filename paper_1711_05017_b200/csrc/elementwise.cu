// elementwise.cu -- the two N^d elementwise steps of the spectral and
// landscape paths that sit between the heavy kernels:
//   * gf_phase_window: C(w) = A(w) exp(2 pi i w.s) over a window in place
//     (spectral.center_window, /root/reference/pkg/src/geofield/
//     spectral.py:184-195: s = the grid centre; also used with other shifts),
//     the phase argument w.s = sum_a (k_a - w_a/2) dw_a s_a summed in float64
//     and reduced to [-1/2, 1/2] cycles before sincospi;
//   * gf_wrap_mask: the landscape's seam mask (energy._wrap_mask,
//     energy.py:286-306) from per-axis flags decided on the host with the
//     reference's float64 compares: mask[i] = OR_a flag_a[i_a].
#include "../../include/geofield_b200.h"
#include "common.cuh"

#include <math.h>

namespace gf {
namespace {

__global__ void phase_window_kernel(cx<double>* __restrict__ data, int w0, int w1, int w2, double t0, double t1,
                                    double t2) {
  const int64_t n = (int64_t)w0 * w1 * w2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(i % w2);
    const int k1 = (int)((i / w2) % w1);
    const int k0 = (int)(i / ((int64_t)w1 * w2));
    double cyc = (double)(k0 - w0 / 2) * t0 + (double)(k1 - w1 / 2) * t1 + (double)(k2 - w2 / 2) * t2;
    cyc -= rint(cyc);
    double s, c;
    sincospi(2.0 * cyc, &s, &c);
    data[i] = data[i] * mk<double>(c, s);
  }
}

__global__ void wrap_mask_kernel(uint8_t* __restrict__ mask, const uint8_t* __restrict__ flags, int n0, int n1,
                                 int n2) {
  const int64_t n = (int64_t)n0 * n1 * n2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(i % n2);
    const int k1 = (int)((i / n2) % n1);
    const int k0 = (int)(i / ((int64_t)n1 * n2));
    mask[i] = flags[k0] | flags[n0 + k1] | flags[n0 + n1 + k2];
  }
}

}  // namespace
}  // namespace gf

using namespace gf;

extern "C" int gf_phase_window(void* data_c128, int d, const int32_t* w, const double* domega, const double* shift,
                               void* stream) {
  GF_CHECK(data_c128 && w && domega && shift && (d == 2 || d == 3), GF_EINVAL, "bad argument");
  int ww[3] = {1, 1, 1};
  double t[3] = {0.0, 0.0, 0.0};
  for (int a = 0; a < d; ++a) {
    ww[a] = w[a];
    t[a] = domega[a] * shift[a];
  }
  const int64_t n = (int64_t)ww[0] * ww[1] * ww[2];
  if (n == 0) return 0;
  int grid = (int)ceil_div(n, 256);
  if (grid > sm_count() * 16) grid = sm_count() * 16;
  phase_window_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(reinterpret_cast<cx<double>*>(data_c128), ww[0], ww[1],
                                                               ww[2], t[0], t[1], t[2]);
  GF_CUDA(cudaGetLastError());
  return 0;
}

extern "C" int gf_wrap_mask(uint8_t* mask_dev, int d, const int32_t* dims, const uint8_t* axis_flags, void* stream) {
  GF_CHECK(mask_dev && dims && axis_flags && (d == 2 || d == 3), GF_EINVAL, "bad argument");
  int nn[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) nn[a] = dims[a];
  const int64_t n = (int64_t)nn[0] * nn[1] * nn[2];
  if (n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nf = (size_t)nn[0] + nn[1] + nn[2];
  uint8_t host[3 * 1024 + 3];
  GF_CHECK(nf <= sizeof host, GF_EINVAL, "axis longer than 1024");
  size_t o = 0;
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < nn[a]; ++i) host[o++] = a < d ? axis_flags[(a == 0 ? 0 : (a == 1 ? nn[0] : nn[0] + nn[1])) + i] : 0;
  void* f = nullptr;
  GF_CUDA(cudaMallocAsync(&f, nf, st));
  GF_CUDA(cudaMemcpyAsync(f, host, nf, cudaMemcpyHostToDevice, st));
  int grid = (int)ceil_div(n, 256);
  if (grid > sm_count() * 16) grid = sm_count() * 16;
  wrap_mask_kernel<<<grid, 256, 0, st>>>(mask_dev, (const uint8_t*)f, nn[0], nn[1], nn[2]);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(f, st);
  GF_CUDA(e);  // (a pageable H2D copy returns once `host` is staged: no sync needed)
  return 0;
}
