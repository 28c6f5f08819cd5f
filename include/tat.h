/*
 * tat.h -- C ABI of libtat: the fast O(n^2 log n) 2-D circular-geometry wave operators
 * of arxiv 2510.24687 ("PAT/TAT"), forward A and exact adjoint A*, on one B200 (sm_100a).
 *
 * Operation (§3.1 Algorithm 1; §3.2 Algorithm 2):
 *   A  : initial pressure f on an n x n grid  ->  traces g(t_m, z_d) at detectors z_d on the
 *        circle of radius R (E:green_conv, L210-216; discretised as DESIGN.md "D0-D7").
 *   A* : the exact transpose of the discrete A under the L2 inner products of
 *        eqn:innerProducts (L217-222):  A* = omega * A^T,
 *        omega = dt * 2 pi R / (n_ring * h^2)  (readings G4, G18, G20).
 *
 * Conventions:
 *   - f[b][iy][ix] (float32, row-major, contiguous) is the sample at
 *       x = (ix - n/2) h, y = (iy - n/2) h, h = 2/n          (reading G1)
 *   - g[b][m][d] (float32, row-major, contiguous) is the trace at t_m = (m+1) T / n_t
 *       (reading G2) and detector d, in the caller's detector_angles order.
 *   - detector_angles are radians, counter-clockwise from +x.  When they lie on a canonical
 *       uniform ring theta = 2 pi r / n_ring (reading G3; n_ring = the smallest multiple of 4
 *       >= n_det fitting every angle within 1e-9 rad) the angular synthesis/analysis are ring
 *       FFTs; otherwise (dense mode, reading G24) n_ring = n_phi = the smallest power of two
 *       >= max(n_det, 8) and the synthesis/analysis are dense sums at the exact angles,
 *       run as 3xTF32 tcgen05 GEMMs (fp32-level accuracy; TAT_DENSE_TC=0 at plan creation
 *       selects the exact-fp32 SIMT kernels, =2 the SIMT analysis only; debugging)
 *       (tat_inverse is not available in dense mode).
 *   - Every call processes exactly `batch` images (the batch the plan was created for).
 *
 * Ownership: the plan owns its device tables and its workspace (allocated at create time).
 * The caller owns f, g and the stream.  tat_forward / tat_adjoint only ENQUEUE kernels on
 * `stream`: no host synchronisation, no allocation, no memcpy; asynchronous faults surface
 * at the caller's next synchronisation.  Calls on one plan must be stream-ordered (the
 * workspace is shared); distinct plans are independent.
 *
 * Errors: arguments are validated on the host before any launch; a failed call writes
 * nothing.  The thread-local message of the last failure is tat_last_error().
 * NaN/Inf in f or g propagate (no scan pass).
 *
 * Alignment: every DEVICE buffer passed to an entry point (f, g, g_obs, r, roi, ...) must be
 * 16-byte aligned (the kernels move it with bulk copies, TMA and 16-byte vector accesses);
 * an unaligned pointer is rejected with TAT_ERR_INVALID_ARGUMENT before any launch.  Host
 * buffers of the *_host variants have no alignment requirement.
 *
 * CUDA graphs: every entry point except tat_plan_create, tat_power_norm, tat_nnls_converge
 * and a tat_inverse with a new r0 is enqueue-only and may be captured.  A launch copies the
 * plan's operator state (tables, quadrature / interpolation rule) by value into its kernel
 * parameters, so a graph captured before a tat_plan_set_* call that changed the operator keeps
 * applying the OLD operator: recapture after such a call (tat_plan_info_t.generation counts
 * them; a graph is current while the generation it was captured at is unchanged).
 *
 * Kernels of a call are launched with programmatic dependent launch (each kernel's table loads
 * overlap its predecessor's tail); the environment variable TAT_PDL=0, read at plan creation,
 * disables it (debugging).
 */
#ifndef TAT_H
#define TAT_H

#include <stddef.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tat_plan tat_plan;   /* opaque */

typedef enum {
  TAT_OK = 0,
  TAT_ERR_INVALID_ARGUMENT = 1,     /* null pointer, n < 8 / odd / not a power of two, n_det < 1,
                                       n_t < 1, batch < 1, R, c, T not finite > 0, non-finite angle */
  TAT_ERR_UNSUPPORTED_GEOMETRY = 2, /* two detectors on one ring position, or a size the
                                       sm_100a kernels do not implement (see tat_last_error()) */
  TAT_ERR_OUT_OF_MEMORY = 3,
  TAT_ERR_CUDA = 4                  /* CUDA API or launch failure */
} tat_status;

/* Build a plan (the Bessel values J_|k|(R lambda_j) are
 * precomputed; here in float64 on the host by Miller's downward recurrence, then stored as
 * float32 multiplier tables on the device together with the bilinear resampling tables).
 *   plan            out: *plan receives the new plan (unchanged on failure)
 *   n               image side (even power of two; kernels implement 32 <= n <= 1024)
 *   n_det, n_t      detectors and time samples
 *   R, c, T         ring radius, speed of sound, time horizon (t in (0, T])
 *   batch           images per call
 *   detector_angles host array of n_det float64 radians (copied; caller keeps ownership)
 * Synchronous (uses the legacy default stream for uploads).  Errors as above. */
tat_status tat_plan_create(tat_plan** plan, int n, int n_det, int n_t,
                           double R, double c, double T, int batch,
                           const double* detector_angles);

/* g = A f  (Algorithm 1).  f: device [batch][n][n] float32; g: device [batch][n_t][n_det]
 * float32.  Enqueued on `stream`.  TAT_ERR_INVALID_ARGUMENT on null plan/pointers. */
tat_status tat_forward(const tat_plan* plan, const float* f, float* g, cudaStream_t stream);

/* f = A* g  (Algorithm 2 as the exact transposed chain).  g: device [batch][n_t][n_det];
 * f: device [batch][n][n].  Enqueued on `stream`. */
tat_status tat_adjoint(const tat_plan* plan, const float* g, float* f, cudaStream_t stream);

/* Host-buffer variants (end-to-end path): copy the host input into plan-owned device staging
 * (cudaMemcpyAsync on `stream`), run the operator, copy the result back to the host buffer.
 * Stream-ordered: the caller synchronises `stream` before reading the output.  Pinned host
 * memory gives asynchronous copies; pageable memory is staged by the driver. */
tat_status tat_forward_host(const tat_plan* plan, const float* f_host, float* g_host,
                            cudaStream_t stream);
tat_status tat_adjoint_host(const tat_plan* plan, const float* g_host, float* f_host,
                            cudaStream_t stream);

/* Pipelined host-buffer pair (the end-to-end path of bench.py): g = A f, u = A* g for host
 * buffers f_host [batch][n][n], u_host [batch][n][n] and optionally g_host [batch][n_t][n_det]
 * (NULL: g stays on the device).  The plan owns two device staging sets and two copy streams:
 * the H2D copy of call i runs on the plan's input stream, the operators on `stream`, the D2H
 * copies on the plan's output stream, so call i's copies overlap the compute of calls i-1 and
 * i+1 (pinned host memory is required for the overlap; pageable memory works, serialised).
 * Call i's host buffers may be reused once it has completed; tat_host_join(plan, s) makes
 * stream s wait for every copy enqueued so far (synchronise s afterwards to read the results).
 * The first call after a join (or ever) is also ordered after the work already on `stream`.
 * Not capturable (uses plan-internal streams).  Errors as tat_forward. */
tat_status tat_pair_host(const tat_plan* plan, const float* f_host, float* g_host, float* u_host,
                         cudaStream_t stream);
tat_status tat_host_join(const tat_plan* plan, cudaStream_t stream);

/* ---- Inverse: A^{-1} g by the approximate universal backprojection of
 * PAPER.md §3.3 Algorithm 3 (L703-784): analysis of g on the ring, the sine transform and the
 * multiplier -2 (-i)^|k| J'_|k|(lambda) (E:Four_coef_v with the 2 pi of reading G21 removed),
 * angular synthesis, bilinear interpolation in (lambda, phi) to the Cartesian nodes inside
 * |xi| < lambda_max, the inverse 2-D DFT, the constant C of E:silly_integral over the annulus
 * r0 < |x| < R, and Pi_Omega0 = restriction to |x| <= r0 (readings G22, G23).
 *   g  device [batch][n_t][n_det];  f  device [batch][n][n] (output);  0 < r0 < R.
 * The paper derives A^{-1} for R = c = 1: other R, c return TAT_ERR_UNSUPPORTED_GEOMETRY.
 * The first call builds the interpolation tables (synchronous, ~32 bytes per Cartesian node of
 * the half spectrum); a call with a new r0 uploads a pixel mask (synchronous); otherwise
 * enqueue-only on `stream`. */
tat_status tat_inverse(const tat_plan* plan, const float* g, float* f, double r0,
                       cudaStream_t stream);

/* ---- Quadrature in lambda (DESIGN reading G25).  PAPER.md L510-513 asks
 * for "a quadrature rule with discretization points clustering toward lambda = 0" for the
 * harmonics k in {-1, 0, 1} without a law; the default is the uniform trapezoid for every k
 * (reading G9), whose k = 0 endpoint error is the t-independent offset -(dlam^2/12) fhat_0(0).
 *   TAT_QUAD_TRAPEZOID  the base definition (default).
 *   TAT_QUAD_LOWK       adds the trapezoid's Euler-Maclaurin endpoint term at lambda = 0, what a
 *                       rule clustering at 0 converges to: A f gains (dlam^2/12)(h^2/2pi) sum f
 *                       on every sample (k = +-1 need no term at this order), A* the adjoint
 *                       omega (dlam^2/12)(h^2/2pi) sum g on every pixel; one extra reduction
 *                       kernel per call, added in the last kernel's epilogue.
 * Applies to tat_forward / tat_adjoint and everything built on them (scaled forward, transpose,
 * residual, adjoint step, NNLS, power norm); tat_inverse is unaffected.  Not thread-safe with
 * calls in flight on the plan (the per-image constants live in the plan's workspace). */
#define TAT_QUAD_TRAPEZOID 0
#define TAT_QUAD_LOWK 1
tat_status tat_plan_set_quadrature(tat_plan* plan, int rule);

/* ---- Cartesian -> polar interpolation (DESIGN reading G26; not in the
 * paper).  Bilinear interpolation on the frequency grid of pitch pi/L samples, to leading order,
 * the transform of K f with K(x) = sinc^2(x1/2L) sinc^2(x2/2L), sinc(u) = sin(pi u)/(pi u).
 *   TAT_INTERP_BILINEAR  the paper's rule (default).
 *   TAT_INTERP_DEAPOD    A_D = A D, D = diag(1/K) on the pixel nodes x_i = (i - n/2) h: K1 scales
 *                        its input rows, and A_D* = D A* (K1T's epilogue).  No extra launches.
 * Same scope and caveats as tat_plan_set_quadrature (tat_inverse unaffected); the two combine
 * (the G25 term is then taken on D f). */
#define TAT_INTERP_BILINEAR 0
#define TAT_INTERP_DEAPOD 1
tat_status tat_plan_set_interpolation(tat_plan* plan, int rule);

/* ---- Euclidean transposes for reverse-mode autodiff.  A* is the L2
 * adjoint omega A^T (reading G20); a framework's backward pass needs the Euclidean transpose:
 *   d/df <A f, w>  = A^T w      -> tat_transpose(g = w, f = out):  out = A^T w = A* w / omega
 *   d/dg <A* g, v> = omega A v  -> tat_forward_scaled(f = v, g = out, alpha = omega)
 * tat_forward_scaled: g = alpha * A f (alpha applied in the last forward kernel).
 * Shapes, streams and errors as tat_forward / tat_adjoint; alpha must be finite. */
tat_status tat_transpose(const tat_plan* plan, const float* g, float* f, cudaStream_t stream);
tat_status tat_forward_scaled(const tat_plan* plan, const float* f, float* g, float alpha,
                              cudaStream_t stream);

/* ---- Iterative reconstruction driver.  NNLS as projected gradient descent,
 * PAPER.md §4.2 "Reconstruction methods" L838-850 (E:operators L164-167):
 *     f^(k+1/2) = f^(k) - lambda A*(A f^(k) - g),   f^(k+1) = Pi_Omega0 max(0, f^(k+1/2))
 * (eq:NNLS-projstep, eqn:projectionHalfCircle).  The residual and the update are fused into
 * the epilogues of the last forward / adjoint kernels (no extra elementwise passes).
 *
 * tat_residual:     r = A f - g_obs.  f device [batch][n][n]; g_obs, r device
 *                   [batch][n_t][n_det] (r may not alias g_obs).  Enqueued on `stream`.
 * tat_adjoint_step: f <- P(f - lambda A* r) in place, P = max(0, .) if nonneg != 0, then times
 *                   roi[iy][ix] (device [n][n] float32 mask, shared by the batch) if roi != NULL.
 *                   TAT_ERR_INVALID_ARGUMENT if lambda is not finite.
 * tat_nnls:         `iters` iterations of the two calls above (r_work: device data-sized
 *                   scratch).  f holds the start value (the paper starts from 0) and receives
 *                   the iterate.  Enqueue-only: capturable in a CUDA graph.
 * tat_power_norm:   lambda_max = the largest eigenvalue of A*A (Rayleigh quotients of `iters`
 *                   power iterations from a seeded counter-based random start over the whole
 *                   batch); the step lambda of eq. NNLS must satisfy 0 < lambda < 2 / lambda_max.
 *                   SYNCHRONOUS (setup): synchronises `stream`; uses plan-owned buffers. */
tat_status tat_residual(const tat_plan* plan, const float* f, const float* g_obs, float* r,
                        cudaStream_t stream);
tat_status tat_adjoint_step(const tat_plan* plan, const float* r, float* f, float lambda,
                            int nonneg, const float* roi, cudaStream_t stream);
tat_status tat_nnls(const tat_plan* plan, const float* g_obs, float* f, float* r_work,
                    float lambda, int iters, int nonneg, const float* roi, cudaStream_t stream);
tat_status tat_power_norm(const tat_plan* plan, int iters, unsigned long long seed,
                          double* lambda_max, cudaStream_t stream);

/* tat_nnls_converge: the same iteration with the paper's stopping criterion (§4.3
 * L968-971: "the L2 norm of an update to the current approximation is smaller than 0.3% of the
 * L2 norm of the very first (non-zero) approximation"; DESIGN reading G28), per image:
 *   the first iterate k0 >= 1 with ||f^k0|| > 0 sets the scale s_b = ||f^k0||_2 (no test on it);
 *   image b stops after the first CHECKED iteration k > k0 with ||f^k - f^(k-1)||_2 < rel_tol s_b
 *   (the paper's rel_tol = 3e-3); its iterate is then frozen while the other images go on.
 * Iterations are checked while some image has no scale yet and then every `check_every`-th
 * (k % check_every == 0; 1 = every iteration, the paper's rule exactly).  Each check is one
 * deterministic device reduction (fixed-order float64 partials) read by the host.
 *   iters_out  host [batch]: iterations applied to image b (= the stopping k), or -max_iters if
 *              the rule was not met within max_iters.
 * SYNCHRONOUS (host loop; synchronises `stream` at every check).  max_iters, check_every >= 1,
 * rel_tol > 0; other arguments as tat_nnls. */
tat_status tat_nnls_converge(const tat_plan* plan, const float* g_obs, float* f, float* r_work,
                             float lambda, int max_iters, int check_every, double rel_tol, int nonneg,
                             const float* roi, int* iters_out, cudaStream_t stream);

/* NULL-safe.  The caller must ensure no work using the plan is in flight. */
void tat_plan_destroy(tat_plan* plan);

/* Introspection: the plan's derived constants (D0) and table sizes. */
typedef struct {
  int n, n_det, n_t, batch;
  int N;            /* Cartesian FFT size 2L/h */
  int J;            /* last radial index; N_lambda = J + 1 */
  int M;            /* DCT-I length; the lambda->t transform runs as a 2M-point FFT */
  int n_ring;       /* canonical ring size = n_phi (dense mode: the polar grid's n_phi) */
  int K;            /* n_ring / 2; harmonics k in [-K, K-1] */
  int n_nodes_half; /* polar nodes in the half-plane store (n_ring/2 * (J+1)) */
  double L, T_new, dxi, dlam, omega, dt, h, wJ;
  size_t workspace_bytes, table_bytes;
  int launches_forward, launches_adjoint;
  int n_targets;    /* Cartesian targets of the transposed bilinear (half spectrum, per image) */
  unsigned generation; /* operator changes by tat_plan_set_* since creation (graph currency) */
} tat_plan_info_t;

/* ring_index: optional host int array of n_det receiving the ring position r_d of each
 * detector (or NULL). */
tat_status tat_plan_info(const tat_plan* plan, tat_plan_info_t* out, int* ring_index);

/* Host-only (no device access): validate the arguments exactly as tat_plan_create does and
 * report the derived constants.  Returns TAT_ERR_UNSUPPORTED_GEOMETRY (with `out` filled)
 * when the geometry is valid but outside what the sm_100a kernels implement. */
tat_status tat_plan_derive(int n, int n_det, int n_t, double R, double c, double T, int batch,
                           const double* detector_angles, tat_plan_info_t* out, int* ring_index);

/* Host-only: the float32 multiplier table the plan uploads, row-major [K+1][J+1]:
 *   m'[k][j] = (h^2/2pi) (1/n_ring) w_j dlam lambda_j J_k(R lambda_j)
 * (E:eq2 P:L463-466 with the trapezoid rule in lambda and the 1/n_phi of E:eq3 and the
 * h^2/2pi of the F_2D convention folded in).  out_len is in floats. */
tat_status tat_plan_host_multiplier(int n, int n_det, int n_t, double R, double c, double T,
                                    const double* detector_angles, float* out, size_t out_len);

/* Optional per-stage device timing (CUDA events recorded between the kernels of each call on
 * the call's stream).  tat_profile_begin arms recording for up to max_calls calls;
 * tat_profile_end synchronises the events and writes the summed milliseconds per stage:
 * stage_ms[0..4] = forward K1..K5, stage_ms[5..10] = adjoint K5T, K4T, K3T, K2Ta (target
 * sums), K2Tb (inverse column transforms), K1T (11 floats), and the number of forward /
 * adjoint calls recorded.  Not thread-safe with concurrent calls. */
tat_status tat_profile_begin(tat_plan* plan, int max_calls);
tat_status tat_profile_end(tat_plan* plan, float* stage_ms, int* n_forward, int* n_adjoint);

const char* tat_status_string(tat_status s);
const char* tat_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TAT_H */
