// fft.cu -- batched line FFTs along one axis of a 3D array (stages 2 and 4).
//
// The reference computes its spectra with numpy's pocketfft
// (spectral.forward_dft / inverse_dft, spectral.py:114-130; the landscape's
// inverse, energy.py:343).  Here each pass transforms every line of one axis
// in shared memory with a radix-2 Stockham FFT (natural order in and out),
// and folds in the index bookkeeping the reference does with
// fftshift / ifftshift / truncation and per-axis phase ramps:
//
//   input  element i of a line sits at FFT position
//            i                      (node order, in_centered = 0)
//            (i - Lin/2) mod N      (DC-centred window of Lin modes, zero-padded)
//          and is multiplied by exp(2 pi i m in_phase), m its mode number;
//   output element i reads FFT position
//            i                      (node order)
//            (i - Lout/2) mod N     (DC-centred window of Lout modes: truncation)
//          times exp(2 pi i m out_phase) * scale.
//
// So a forward centred window C = dV fftshift(fftn(ifftshift f))[window] is
// three passes with out_phase = 1/2 ((-1)^m) and only Lout = w outputs per
// line written: every later pass reads w/N of the previous volume.  The
// landscape's zero-padded inverse reads only the w^d window (in_centered).
//
// Tile: one CTA owns B lines of length N.  For the contiguous axis the B
// lines are consecutive in memory; for the other axes the B lines are B
// consecutive positions of the last axis -- in both cases global loads and
// stores are coalesced.  Twiddles come from a per-CTA shared table built
// with sincospi (float64).
#include "../../include/geofield_b200.h"
#include "common.cuh"

#include <math.h>

namespace gf {
namespace {

struct FftArgs {
  const void* in;
  void* out;
  int shape_in[3];
  int shape_out[3];
  int axis;
  int N;
  int in_centered, out_centered;
  int sign;  // -1 forward, +1 inverse
  double in_phase, out_phase, scale;
  int B;     // lines per CTA
};

template <typename T>
__global__ void __launch_bounds__(256) fft_lines_kernel(FftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = a.N, B = a.B, half = N >> 1;
  const int ld = N + 1;  // padded line stride (complex elements)
  cx<T>* buf0 = reinterpret_cast<cx<T>*>(smem_raw);
  cx<T>* buf1 = buf0 + B * ld;
  cx<T>* tw = buf1 + B * ld;  // N/2 twiddles
  const int ax = a.axis;
  const int Lin = a.shape_in[ax], Lout = a.shape_out[ax];
  const int tid = threadIdx.x, nt = blockDim.x;

  for (int k = tid; k < half; k += nt) {
    double s, c;
    sincospi((double)a.sign * 2.0 * (double)k / (double)N, &s, &c);
    tw[k] = mk<T>((T)c, (T)s);
  }

  // line tile decode: shapes (s0, s1, s2); contiguous axis 2
  const int s2i = a.shape_in[2];
  int64_t base_in, base_out, stride_in, stride_out, lstep_in, lstep_out;
  int nlines;  // lines in this tile
  if (ax == 2) {
    const int64_t lines = (int64_t)a.shape_in[0] * a.shape_in[1];
    const int64_t l0 = (int64_t)blockIdx.x * B;
    nlines = (int)min((int64_t)B, lines - l0);
    base_in = l0 * Lin;
    base_out = l0 * Lout;
    stride_in = 1;
    stride_out = 1;
    lstep_in = Lin;
    lstep_out = Lout;
  } else {
    // lines = other-axis index o (size so) x last-axis position p (size s2)
    const int so = ax == 0 ? a.shape_in[1] : a.shape_in[0];
    const int ptiles = (s2i + B - 1) / B;
    const int o = blockIdx.x / ptiles, p0 = (blockIdx.x % ptiles) * B;
    nlines = min(B, s2i - p0);
    (void)so;
    if (ax == 0) {  // element (j, o, p): ((j * s1 + o) * s2 + p)
      base_in = (int64_t)o * s2i + p0;
      base_out = (int64_t)o * a.shape_out[2] + p0;
      stride_in = (int64_t)a.shape_in[1] * s2i;
      stride_out = (int64_t)a.shape_out[1] * a.shape_out[2];
    } else {        // ax == 1, element (o, j, p)
      base_in = (int64_t)o * a.shape_in[1] * s2i + p0;
      base_out = (int64_t)o * a.shape_out[1] * a.shape_out[2] + p0;
      stride_in = s2i;
      stride_out = a.shape_out[2];
    }
    lstep_in = 1;
    lstep_out = 1;
  }
  const cx<T>* __restrict__ in = reinterpret_cast<const cx<T>*>(a.in);
  cx<T>* __restrict__ out = reinterpret_cast<cx<T>*>(a.out);

  // zero-fill then scatter the inputs to their FFT positions
  for (int e = tid; e < B * ld; e += nt) buf0[e] = mk<T>(0, 0);
  __syncthreads();
  const int hin = a.in_centered ? Lin / 2 : 0;
  for (int e = tid; e < nlines * Lin; e += nt) {
    int b, j;
    if (ax == 2) { b = e / Lin; j = e % Lin; }
    else { j = e / nlines; b = e % nlines; }
    cx<T> v = in[base_in + (int64_t)b * lstep_in + (int64_t)j * stride_in];
    const int m = j - hin;  // mode number (node index when not centred)
    if (a.in_phase != 0.0) {
      double cyc = a.in_phase * (double)m;
      cyc -= rint(cyc);
      double s, c;
      sincospi(2.0 * cyc, &s, &c);
      v = v * mk<T>((T)c, (T)s);
    }
    const int pos = a.in_centered ? ((m % N) + N) % N : j;
    buf0[b * ld + pos] = v;
  }
  __syncthreads();

  // radix-2 Stockham: span Ns = 1, 2, ..., N/2
  cx<T>* x = buf0;
  cx<T>* y = buf1;
  for (int Ns = 1; Ns < N; Ns <<= 1) {
    const int tstep = N / (2 * Ns);
    for (int e = tid; e < B * half; e += nt) {
      const int b = e / half, j = e % half;
      const int k = j & (Ns - 1);
      const cx<T> t = tw[k * tstep];
      const cx<T> u = x[b * ld + j];
      const cx<T> v = x[b * ld + j + half] * t;
      const int idx = ((j - k) << 1) + k;
      y[b * ld + idx] = u + v;
      y[b * ld + idx + Ns] = u - v;
    }
    __syncthreads();
    cx<T>* tmp = x;
    x = y;
    y = tmp;
  }

  const int hout = a.out_centered ? Lout / 2 : 0;
  for (int e = tid; e < nlines * Lout; e += nt) {
    int b, j;
    if (ax == 2) { b = e / Lout; j = e % Lout; }
    else { j = e / nlines; b = e % nlines; }
    const int m = j - hout;
    const int pos = a.out_centered ? ((m % N) + N) % N : j;
    cx<T> v = x[b * ld + pos];
    double cyc = a.out_phase * (double)m;
    cyc -= rint(cyc);
    double s, c;
    sincospi(2.0 * cyc, &s, &c);
    v = v * mk<T>((T)(c * a.scale), (T)(s * a.scale));
    out[base_out + (int64_t)b * lstep_out + (int64_t)j * stride_out] = v;
  }
}

template <typename T>
cudaError_t launch_fft_pass(FftArgs a, cudaStream_t st) {
  const int N = a.N;
  // lines per CTA: keep two ping-pong buffers + twiddles within ~96 KB
  int B = (int)(96 * 1024 / (2 * (N + 1) * sizeof(cx<T>)));
  if (B > 32) B = 32;
  if (B < 1) B = 1;
  if (a.axis != 2 && B > a.shape_in[2]) B = a.shape_in[2];
  a.B = B;
  size_t smem = (size_t)(2 * B * (N + 1) + N / 2) * sizeof(cx<T>);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(fft_lines_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  int64_t blocks;
  if (a.axis == 2) {
    blocks = ceil_div((int64_t)a.shape_in[0] * a.shape_in[1], B);
  } else {
    const int so = a.axis == 0 ? a.shape_in[1] : a.shape_in[0];
    blocks = (int64_t)so * ceil_div(a.shape_in[2], B);
  }
  fft_lines_kernel<T><<<(unsigned)blocks, 256, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace
}  // namespace gf

using namespace gf;

extern "C" int gf_fft_pass(int precision, const void* in, void* out, const int32_t* shape_in,
                           const int32_t* shape_out, int axis, int n, int in_centered, int out_centered, int sign,
                           double in_phase, double out_phase, double scale, void* stream) {
  GF_CHECK(in && out && shape_in && shape_out, GF_EINVAL, "null argument");
  GF_CHECK(axis >= 0 && axis < 3, GF_EINVAL, "axis must be 0, 1 or 2");
  GF_CHECK(n >= 2 && n <= 4096 && (n & (n - 1)) == 0, GF_EINVAL, "FFT length must be a power of two in [2, 4096]");
  GF_CHECK(sign == -1 || sign == 1, GF_EINVAL, "sign must be -1 or +1");
  GF_CHECK(precision == 32 || precision == 64, GF_EINVAL, "precision must be 32 or 64");
  for (int a = 0; a < 3; ++a)
    if (a != axis) GF_CHECK(shape_in[a] == shape_out[a], GF_EINVAL, "non-transform axes must match");
  GF_CHECK(shape_in[axis] <= n && shape_out[axis] <= n, GF_EINVAL, "line longer than the FFT length");
  GF_CHECK(in_centered || shape_in[axis] == n, GF_EINVAL, "node-ordered input must have length n");
  GF_CHECK(out_centered || shape_out[axis] == n, GF_EINVAL, "node-ordered output must have length n");
  FftArgs a = {};
  a.in = in;
  a.out = out;
  for (int k = 0; k < 3; ++k) {
    a.shape_in[k] = shape_in[k];
    a.shape_out[k] = shape_out[k];
  }
  a.axis = axis;
  a.N = n;
  a.in_centered = in_centered;
  a.out_centered = out_centered;
  a.sign = sign;
  a.in_phase = in_phase;
  a.out_phase = out_phase;
  a.scale = scale;
  cudaStream_t st = (cudaStream_t)stream;
  if (precision == 64) GF_CUDA(launch_fft_pass<double>(a, st));
  else GF_CUDA(launch_fft_pass<float>(a, st));
  return 0;
}
