/*
 * geofield_b200.h -- C ABI of the B200 engine for the geofield hot path.
 *
 * This is the drop-in boundary: a reference-side binding (ctypes, see
 * INTEGRATION.md) replaces the compiled kernels that the reference's operator
 * layer `geofield.backend` dispatches to (/root/reference/pkg/src/geofield/
 * backend.py:71-164 -> _core.pyx).  Plain pointers and sizes only; no torch
 * types.  Every function returns 0 on success, a cudaError_t (> 0) on a CUDA
 * failure, or a negative gf status (-1 bad argument, -2 out of host memory,
 * -3 internal, -4 haptic server no longer running); gf_last_error() then
 * describes the failure (thread-local).
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

/* Density construction (stage 1) ------------------------------------------ */

/* Element arrays: 3D triangles (ne x 9 doubles: v0, v1, v2), 2D segments
 * (ne x 4: a, b); normals (ne x d, outward, unit); measures (ne: triangle
 * areas / segment lengths).  Points P: m x d doubles.  Host in / host out.
 * All float64 with every operation separately rounded (bit-exact distances
 * and decisions against the reference). */

/* Exact min point-element distance and winding number per point; either
 * output may be NULL.  Replaces _core.distance_{2,3}d (_core.pyx:149-230, via
 * backend.distance_batch, backend.py:71-93) and _core.winding_{2,3}d
 * (_core.pyx:262-292, via backend.winding_batch, backend.py:96-113). */
int gf_distance_winding(int d, const double *elems, int64_t ne, const double *P, int64_t m, double *xi_out,
                        double *wind_out);

/* Adaptive skeletal sweep I+ per point.  Replaces _core.sweep_{2,3}d
 * (_core.pyx:300-523) via backend.sweep_batch (backend.py:116-150): out is
 * interleaved complex128 (m), resid (m) is read and max-updated in place,
 * clamps (m) are incremented. */
int gf_sweep(int d, const double *elems, const double *normals, const double *measures, int64_t ne, const double *P,
             const double *xi_eff, int64_t m, double sigma, double gconst, double max_angle, int max_depth,
             double eta_min, double *out_c128, double *resid, int64_t *clamps);

/* Whole affinity_field (descriptor.py:309-357) on the grid nodes, device
 * resident: distance + winding, sweep (family 1 = SkeletalDensity; 0 =
 * InverseSquare, values = winding), combine, neighbour fill of excluded
 * nodes.  values_dev: complex128 node values (device); flags_dev: one byte
 * per node (bit0 excluded, bit1 unresolved, bit2 inside); stats[0] = total
 * eta clamps, stats[1] = worst residual, stats[2] = seconds of the fused
 * distance + winding kernel, stats[3] = seconds of the sweep (device time);
 * `stats` holds 4 doubles. */
int gf_affinity_grid(int d, const double *elems, const double *normals, const double *measures, int64_t ne,
                     const int32_t *dims, const double *origin, double spacing, int family, double sigma,
                     double gconst, double lam_in, double lam_out, double max_angle, int max_depth, double eta_floor,
                     void *values_dev, uint8_t *flags_dev, double *stats, void *stream);

/* Winding number at every node of a grid (dims, origin, spacing as in
 * gf_affinity_grid) into a device array of node_count doubles; the
 * indicator field of descriptor.py:360-366 is wind >= 0.5 (bit-exact). */
int gf_winding_grid(int d, const double *elems, int64_t ne, const int32_t *dims, const double *origin, double spacing,
                    void *wind_dev, void *stream);

/* Slab of the same pipeline for multi-GPU node sharding:
 * owned axis-0 planes [plane0, plane0 + nplanes) of the global grid `dims`,
 * computed together with halo_lo / halo_hi neighbour planes so the
 * excluded-node neighbour fill sees across the slab boundary; node
 * coordinates use the global index (bit-identical to gf_affinity_grid).
 * Outputs hold only the owned planes; stats cover only the owned nodes. */
int gf_affinity_planes(int d, const double *elems, const double *normals, const double *measures, int64_t ne,
                       const int32_t *dims, const double *origin, double spacing, int32_t plane0, int32_t nplanes,
                       int32_t halo_lo, int32_t halo_hi, int family, double sigma, double gconst, double lam_in,
                       double lam_out, double max_angle, int max_depth, double eta_floor, void *values_dev,
                       uint8_t *flags_dev, double *stats, void *stream);

/* Multi-GPU slab exchange fused into an axis-1 pass: the FFT of this
 * rank's lines (shape_in = (nk, L1, N2), length-n transform, input / output
 * node-ordered or DC-centred exactly as gf_fft_pass, out_len rows out) with
 * output row y of plane x stored into rank s's y-slab (planes, ny_s, N2) at
 * plane x_off + x, row y - y_bounds[s] (y_bounds tile [0, out_len));
 * dst_ptrs[s] is that slab's device address (a peer mapping on another GPU,
 * e.g. a symmetric-memory buffer).  Replaces pass + all-to-all in
 * parallel.score_field_slab and forward_window_slab (W1). */
int gf_fft_pass_scatter(int precision, const void *in, const int32_t *shape_in, int n, int in_centered, int out_len,
                        int out_centered, int sign, double in_phase, double out_phase, double scale, int nranks,
                        const int32_t *y_bounds, const uint64_t *dst_ptrs, int x_off, void *stream);

/* Spectra (stage 2) and landscapes (stage 4) ------------------------------ */

/* One batched line-FFT pass along `axis` of a 3D row-major complex array
 * (2D data: shape (1, n0, n1)); precision 32 (complex64) or 64 (complex128),
 * device buffers, stream-ordered.  Input element i of a line sits at FFT
 * position i (in_centered = 0, length n) or (i - Lin/2) mod n (DC-centred
 * window, zero-padded) and is scaled by exp(2 pi i m in_phase); output
 * element i reads position i or (i - Lout/2) mod n (centred truncation) and
 * is scaled by scale * exp(2 pi i m out_phase), m = mode number.  sign -1
 * forward, +1 inverse (unnormalised).  Three passes realise
 * spectral.forward_dft / truncate / center_window / inverse_dft
 * (spectral.py:114-195) and the landscape's zero-padded inverse
 * (energy.py:336-343). */
int gf_fft_pass(int precision, const void *in, void *out, const int32_t *shape_in, const int32_t *shape_out,
                int axis, int n, int in_centered, int out_centered, int sign, double in_phase, double out_phase,
                double scale, void *stream);

/* Q(w) = C1(w) V(w) exp(2 pi i w.s) over the window, V = multilinear sample
 * of window h2 at u = -R^T w / dw + w/2 (zero outside unless wrap; float64
 * floor decisions as the cascade); h1 = 0 means C1 = 1
 * (rotate_reflect_spectrum, spectral.py:204-226).  out_dev: window-shaped,
 * complex64/complex128 by precision. */
int gf_rotate_product(uint64_t h1, uint64_t h2, int wrap, const double *domega, const double *R, const double *s,
                      int precision, void *out_dev, void *stream);

/* Same restricted to window x-planes [kx0, kx0 + nkx) (nkx < 0: all); out
 * is (nkx, w1, w2).  The slab-decomposed landscape gives each rank its own
 * kx-planes. */
int gf_rotate_product_planes(uint64_t h1, uint64_t h2, int wrap, const double *domega, const double *R,
                             const double *s, int precision, int kx0, int nkx, void *out_dev, void *stream);

/* Full translational landscape (energy.score_field, energy.py:309-344):
 * the product above with s = Rc - c + origin, then three pruned inverse
 * passes to the dims grid, times scale (= 1 / (N^d dV)).  work_dev holds
 * >= w N^2 elements, work2_dev >= w^2 N (2D: w, w N), out_dev N^d. */
int gf_score_field(uint64_t h1, uint64_t h2, int wrap, const double *domega, const int32_t *dims, const double *R,
                   const double *s, double scale, int precision, void *work_dev, void *work2_dev, void *out_dev,
                   void *stream);

/* Elementwise steps between the heavy kernels (device buffers, stream-
 * ordered): C *= exp(2 pi i w.s) over a DC-centred complex128 window in
 * place, the phase summed over axes in float64 (spectral.center_window,
 * spectral.py:184-195, with s = the grid centre); and the landscape's seam
 * mask (energy._wrap_mask, energy.py:286-306) as OR of per-axis host flags
 * (dims[0] + dims[1] (+ dims[2]) bytes) into one byte per node. */
int gf_phase_window(void *data_c128, int d, const int32_t *w, const double *domega, const double *shift, void *stream);
int gf_wrap_mask(uint8_t *mask_dev, int d, const int32_t *dims, const uint8_t *axis_flags, void *stream);

/* Moment-spectrum rotational gradient (energy._rotational_gradient_vector,
 * energy.py:210-251): the reference's independent cross-check of the torque
 * from the moving part's centre-referenced moment windows hmom[0..d-1]
 * (the windows of rho p_a).  out receives d_rot interleaved complex128
 * values (3 in 3D, 1 in 2D; the rest zero), already 2 pi i dcell scaled.
 * float64 throughout, one fused pass over the window. */
int gf_vector_torque(uint64_t h1, uint64_t h2, const uint64_t *hmom, int wrap, const double *domega, double dcell,
                     const double *R, const double *t_eff, const double *center, double *out);

/* Diagnostics: FMA-pipe peak (TFLOP/s, 2 flops per FMA) measured with an
 * FMA-chain kernel on the current device; the roofline denominator of the
 * query/sweep kernels (precision 32 or 64). */
int gf_measure_fma_peak(int precision, double *tflops);
/* Launch-overhead probe: host and device microseconds per empty launch. */
int gf_measure_launch(int n, int blocks, double *host_us, double *dev_us);
/* Host<->device round trips (diagnostics for the query path): out[0] launch +
 * mapped completion p50 us, out[1] pre-enqueued kernel released by a mapped
 * flag (cuStreamWaitValue32) p50 us, out[2] GPU read latency of mapped host
 * memory ns, out[3] mapped write + system fence ns. */
int gf_measure_roundtrip(int n, double *out);
/* GPU-wide stall detector: one warp per SM spins on %globaltimer for
 * `seconds` (<= 60) with no host interaction.  out[0] longest gap between
 * consecutive reads on any SM (us), out[1] / out[2] fewest / most gaps over
 * threshold_us on one SM (equal counts on every SM: the whole GPU stopped),
 * out[3] SMs watched. */
int gf_measure_stalls(double seconds, double threshold_us, double *out);

/* Persistent haptic server (Q1 latency path): a resident grid serves one
 * query per call through a host-mapped mailbox -- no kernel launch per
 * query.  Same window pair / grid for the server's lifetime; the kernel exits
 * after idle_timeout_s without requests (<= 0: 30 s) or on gf_server_stop.
 * max_sms > 0 keeps the grid on about that many SMs (whole CTA clusters by
 * SM id; the rest leave at start-up), so landscape exports and sweeps from
 * other threads run beside a session; 0 uses every SM.
 * gf_server_query has gf_cascade's pose and output conventions and returns
 * -4 once the server has stopped or timed out (the caller falls back to
 * gf_cascade). */
int gf_server_start(uint64_t h1, uint64_t h2, int wrap, const double *domega, double dcell, const double *center,
                    int precision, double idle_timeout_s, int max_sms, uint64_t *server_id);
int gf_server_query(uint64_t server_id, const double *R, const double *t_eff, double *out);
int gf_server_stop(uint64_t server_id);
/* Diagnostics of the server's last query, microseconds (-1: not observed):
 * out[0] host time from posting the request to reading the result, out[1]
 * the GPU's detect -> result time (globaltimer), out[2] post -> detect and
 * out[3] result -> host receipt (host realtime clock vs globaltimer: the two
 * differ by a slowly drifting offset, so compare with a typical query),
 * out[4] the host's time to post the request, out[5] the longest stretch
 * between two mailbox polls of the GPU's polling warp, out[6] the longest
 * stretch between two clock reads of a warp beside it (an SM stall). */
int gf_server_last_timing(uint64_t server_id, double *out7);

/* Experiment knobs: the batched sweep's run length along the run axis per
 * thread (0 = auto), and per-CTA phase timestamps (globaltimer ns) of the
 * single-query kernel into a device buffer of >= 8 x blocks uint64 (NULL
 * disables). */
int gf_set_cascade_run_length(int L);
int gf_set_cascade_debug(void *dev_buf);

#ifdef __cplusplus
}
#endif

#endif /* GEOFIELD_B200_H */
