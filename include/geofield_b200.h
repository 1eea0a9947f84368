/*
 * geofield_b200.h -- C ABI of the B200 engine for the geofield hot path.
 *
 * This is the drop-in boundary: a reference-side binding (ctypes, see
 * INTEGRATION.md) replaces the compiled kernels that the reference's operator
 * layer `geofield.backend` dispatches to (/root/reference/pkg/src/geofield/
 * backend.py:71-164 -> _core.pyx).  Plain pointers and sizes only; no torch
 * types.  Every function returns 0 on success, a cudaError_t (> 0) on a CUDA
 * failure, or a negative gf status (-1 bad argument, -2 out of host memory,
 * -3 internal); gf_last_error() then describes the failure (thread-local).
 * Domain validation (rotation checks, grid mismatch, window budgets) stays in
 * the Python host layer with the reference's exception types.
 *
 * Precision argument: 32 = complex64 storage, FP32 arithmetic (the product
 * default, within 1e-4 of the float64 reference); 64 = float64 throughout
 * (the reference's own tight tolerances).  Floor decisions are always taken
 * in float64 reference order.
 *
 * Threading: all entry points are thread-safe.  Each host thread owns a
 * high-priority CUDA stream for single queries; batched and field entry
 * points take the caller's stream (cudaStream_t passed as void*).
 */
#ifndef GEOFIELD_B200_H
#define GEOFIELD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Library / device ------------------------------------------------------- */

/* Select the CUDA device for the calling thread and create its query
 * stream.  Replaces the import-time `_core` availability check
 * (backend.py:19-25). */
int gf_init(int device);
const char *gf_last_error(void);
int gf_version(void);

/* Window handles --------------------------------------------------------- */

/* Upload a centre-referenced window (complex128, row-major, d = 2 or 3,
 * w[0..d-1] sides; w[2] ignored for d = 2).  Replaces the per-call
 * `np.ascontiguousarray(C, complex128)` marshalling of backend.cascade
 * (backend.py:155-156): windows become device-resident, cached per
 * PartAsset/m' exactly like PartAsset._windows (energy.py:103-121). */
int gf_window_create(const double *host_c128, int d, const int32_t *w, uint64_t *handle);
/* Same from a device buffer (complex128) produced on the GPU (stage 2). */
int gf_window_create_device(const void *dev_c128, int d, const int32_t *w, uint64_t *handle, void *stream);
int gf_window_destroy(uint64_t handle);
/* Device address of the raw complex128 window (for diagnostics/tests). */
int gf_window_device_ptr(uint64_t handle, const void **dev_c128);

/* Cascade (Q1) ------------------------------------------------------------ */

/* One query, host in / host out.  Replaces _core.cascade_3d / cascade_2d
 * (_core.pyx:530-724) as called by backend.cascade (backend.py:153-164):
 * same argument meaning and order; out receives 1 + d + n_rot interleaved
 * complex128 values (7 in 3D, 4 in 2D), already scaled by dcell. */
int gf_cascade(uint64_t h1, uint64_t h2, int wrap, const double *domega, double dcell, const double *R,
               const double *t_eff, const double *center, int precision, double *out);

/* Batched pose sweep (Q3): n poses from device memory, each 12 doubles
 * (R row-major 3x3 then t_eff; 2D poses are embedded with R[2][2] = 1),
 * results to device memory, 14 doubles per pose (interleaved complex128 x7;
 * for d = 2 the rotational term is slot 6).  No reference function: the
 * reference loops evaluate() serially (cli.py:349-356). */
int gf_cascade_batch(uint64_t h1, uint64_t h2, int wrap, const double *domega, double dcell,
                     const double *center, int precision, int64_t n, const double *poses_dev, double *out_dev,
                     void *stream);

/* The single-query path applied to n poses one launch at a time, stream-
 * ordered (the serial haptic loop with inputs resident in HBM; capturable
 * into a CUDA graph).  Same layouts as gf_cascade_batch. */
int gf_cascade_serial(uint64_t h1, uint64_t h2, int wrap, const double *domega, double dcell,
                      const double *center, int precision, int64_t n, const double *poses_dev, double *out_dev,
                      void *stream);

/* Diagnostics: FMA-pipe peak (TFLOP/s, 2 flops per FMA) measured with an
 * FMA-chain kernel on the current device; the roofline denominator of the
 * query/sweep kernels (precision 32 or 64). */
int gf_measure_fma_peak(int precision, double *tflops);
/* Launch-overhead probe: host and device microseconds per empty launch. */
int gf_measure_launch(int n, int blocks, double *host_us, double *dev_us);

/* Tuning knobs for experiments: kernel variant (0 = u-space tiled, the
 * default; 1 = direct gather) and the direct variant's run length along kz
 * per thread (0 = auto). */
int gf_set_cascade_variant(int variant);
int gf_set_cascade_tile(int tile);
int gf_set_cascade_run_length(int L);

#ifdef __cplusplus
}
#endif

#endif /* GEOFIELD_B200_H */
