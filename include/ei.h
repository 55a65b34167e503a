/*
 * include/ei.h — C ABI of libei: the B200 (sm_100a) hot path of model-based iterative
 * edge-illumination (EI) tomography, arxiv 2202.08627 (Modregger et al.).
 *
 * One cost+gradient evaluation per optimizer iteration (eq. 5) of the
 * three-map EI model (absorption mu, refractive decrement delta, scattering
 * sigma), in four stages, all hand-written CUDA for sm_100a:
 *   K1  Joseph projection of mu, delta, sigma at every angle (eq. 1)
 *   K2  fused curve model / residual / cost / dS/dP (eq. 2, eq. 4 :74-75,
 *       eq. 5 :79), including the refraction shift z d/dt R[delta]
 *   K3  pixel-driven, atomic-free adjoint R^T of the three gradient sinograms
 *   K4  fixed-order fp64 per-slice cost
 *
 * Conventions (all entry points)
 *   - Arrays are fp32 (cost: fp64, status: int32), C-contiguous, little-endian.
 *   - Device-pointer entry points are asynchronous on `stream` (a cudaStream_t passed as
 *     void*; NULL = the legacy default stream) and never synchronise the host.  Device
 *     arrays are owned by the caller; outputs are caller-allocated.
 *   - Argument errors are returned synchronously before any launch (EI_ERR_*), and no
 *     output is touched.  Numeric conditions in device data are counted in `status`.
 *   - A plan owns its device workspace (allocated in ei_plan_create) and may serve one
 *     in-flight call at a time; distinct plans are independent.
 *   - Geometry (readings R4-R8): pixel centres x_j = (j-(N-1)/2)*pixel
 *     (j = contiguous index), y_i = (i-(N-1)/2)*pixel; detector u_k = (k-(Nd-1)/2)*det_pitch;
 *     the ray (theta, k) is x cos(theta) + y sin(theta) = u_k.
 *   - Units (R3, R4): mask positions, flat-IC centre/width, drift and the refraction shift
 *     are in mask periods; the shift is z * dR[delta]/dt with dt = det_pitch.
 */
#ifndef EI_H
#define EI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    EI_OK = 0,
    EI_ERR_NULL = 1,      /* a required pointer is NULL                                   */
    EI_ERR_SHAPE = 2,     /* S<1, N<2, Nd<3, n_angles<1, M<1, n_maps not 1|3,
                             16 Nd + 4 M > 225280 (Nd <= 14079 for M <= 4), n_angles > 14080,
                             M too large for K2's staging ring (one detector segment's 3 + M
                             rows in 220 KB of shared memory), a sampled flat IC with < 4
                             knots (tests/test_gpu_limits.py runs parity at these limits)   */
    EI_ERR_DOMAIN = 3,    /* pixel/det_pitch/z <= 0 or non-finite, det_pitch < pixel,
                             non-finite angle, lambda < 0 or non-finite                    */
    EI_ERR_RESOURCE = 4,  /* device allocation failed / size overflow (N^2 > 2^30 or
                             n_angles Nd M > 2^30: 32-bit per-slice indices)                */
    EI_ERR_CUDA = 5       /* a CUDA call or kernel launch failed                           */
};

typedef struct ei_geometry {
    int32_t n_slices;   /* S: independent slices                            */
    int32_t n;          /* N: maps are N x N                                               */
    int32_t n_angles;   /* N_theta                                                          */
    int32_t n_det;      /* N_d detector pixels, >= 3 (finite differences need 3)           */
    int32_t n_mask;     /* M mask positions                                                */
    double pixel;       /* dx, map pixel pitch                                              */
    double det_pitch;   /* du, detector pitch; must satisfy du >= dx (<= 2 adjoint taps)   */
    double z;           /* sample-detector distance factor of the shift      */
} ei_geometry;

typedef struct ei_plan ei_plan;   /* opaque: device angle table + workspace               */

/* Create a plan.  angles_rad_host: [n_angles] host fp64 projection angles.
 * The per-angle table (cos, sin, row/column dominance |cos| >= |sin| decided in fp64,
 * reading R5) is built on the host and uploaded; the workspace (packed maps, P and G
 * sinograms, reduction partials) is allocated here and nowhere else on the device path.
 * Returns EI_OK and *out, or an error (then *out = NULL). */
int ei_plan_create(const ei_geometry *geom, const double *angles_rad_host, ei_plan **out);
void ei_plan_destroy(ei_plan *plan);

/* R: Joseph projection (SPEC.md:49 radon_forward).
 * maps [S][n_maps][N][N] device -> sino [S][n_maps][N_theta][N_d] device. n_maps in {1, 3}. */
int ei_project(const ei_plan *plan, const float *maps, int n_maps, float *sino, void *stream);

/* R^T: the exact transpose of ei_project, pixel-driven tent gather (a5).
 * sino [S][n_maps][N_theta][N_d] device -> maps [S][n_maps][N][N] device (overwritten). */
int ei_backproject(const ei_plan *plan, const float *sino, int n_maps, float *maps, void *stream);

/* Forward model s_mod (SPEC.md:206 forward; eq. 2/4 with m_r = 0, scattering per R1):
 *   mu, delta, sigma [S][N][N]; flat [S][3][N_d] = (A, c, w) of the Gaussian flat IC (R2);
 *   mask_pos [M]; drift [N_theta] = m_o(theta) or NULL (zeros, R14)
 *   -> s_mod [S][N_theta][M][N_d].  All device pointers. */
int ei_forward(const ei_plan *plan, const float *mu, const float *delta, const float *sigma,
               const float *flat, const float *mask_pos, const float *drift, float *s_mod,
               void *stream);

/* Cost and gradient (SPEC.md:261 cost + :270 grad, map blocks), eq. 5:
 *   S_s = sum_{theta,t,m} (s_mod - s_exp)^2 + lambda * sum (mu^2 + delta^2 + sigma^2)
 *   s_exp [S][N_theta][M][N_d]; lambda >= 0 (paper: 1e-2)
 *   -> cost [S] fp64 device; g_mu, g_delta, g_sigma [S][N][N] device (overwritten);
 *      status [4] int32 device, ACCUMULATED (caller zeroes it):
 *        [0] non-finite input elements (maps, flat, mask, drift, s_exp)
 *        [1] (s,theta,t) where P_mu was clamped to [-50, 50] (R12)
 *        [2] (s,theta,t) where W^2 was clamped to w^2/100 (R13)
 *        [3] reserved (0)
 * Exactly one projection and one adjoint per map per call. */
int ei_cost_grad(const ei_plan *plan, const float *mu, const float *delta, const float *sigma,
                 const float *flat, const float *mask_pos, const float *drift, const float *s_exp,
                 float lambda, double *cost, float *g_mu, float *g_delta, float *g_sigma,
                 int32_t *status, void *stream);

/* ei_cost_grad plus the gradient with respect to the mask drift m_o(theta) (SURVEY.md §8(f)
 * NEXT-2; m_o enters eq. 4, through u = m - c - m_o - Delta), computed in the same
 * pass (one extra fixed-order reduction, no extra launch):
 *   g_drift [S][N_theta] fp32 device (overwritten): dS_s/dm_o(theta) of each slice s; the drift
 *   is shared by the slices of a stack, so its gradient is the sum over s (left to the caller, and
 *   across ranks for a slice-sharded stack).  Must not be NULL (EI_ERR_NULL).
 * All other arguments, outputs and errors exactly as ei_cost_grad; a NULL drift means m_o = 0
 * and the gradient is still evaluated there. */
int ei_cost_grad_drift(const ei_plan *plan, const float *mu, const float *delta, const float *sigma,
                       const float *flat, const float *mask_pos, const float *drift,
                       const float *s_exp, float lambda, double *cost, float *g_mu, float *g_delta,
                       float *g_sigma, float *g_drift, int32_t *status, void *stream);

/* The paper's own single-map model: eq. 4 with
 * m_r = 0 under the homogeneity assumption mu = gamma^-1 delta = h,
 * so one projection and one adjoint per evaluation instead of three:
 *   s_mod = exp(-R[h]) * f(t, m - m_o(theta) - z gamma dR[h]/dt)   (no scattering: W = w)
 *   S_s   = sum (s_mod - s_exp)^2 + lambda sum h^2                  (eq. 5; paper gamma = 5,
 *                                                                     lambda = 1e-2)
 * h [S][N][N] device; gamma finite (EI_ERR_DOMAIN otherwise); the plan's geometry (z, pixel,
 * det_pitch, M) as for the three-map model; flat, mask_pos, drift, s_exp as for ei_cost_grad.
 * ei_forward_h -> s_mod [S][N_theta][M][N_d].
 * ei_cost_grad_h -> cost [S] fp64, g_h [S][N][N] (overwritten), g_drift [S][N_theta] or NULL
 * (dS_s/dm_o(theta), as ei_cost_grad_drift), status [4] accumulated: [0] non-finite inputs,
 * [1] P_h clamp hits (R12), [2] 0, [3] 0.  Same conventions as ei_cost_grad otherwise. */
int ei_forward_h(const ei_plan *plan, const float *h, float gamma, const float *flat,
                 const float *mask_pos, const float *drift, float *s_mod, void *stream);
int ei_cost_grad_h(const ei_plan *plan, const float *h, float gamma, const float *flat,
                   const float *mask_pos, const float *drift, const float *s_exp, float lambda,
                   double *cost, float *g_h, float *g_drift, int32_t *status, void *stream);

/* The single-map model with the MEASURED (sampled) flat-field IC: the
 * paper scans the sample mask over one period in 33 steps and evaluates f at the
 * shifted argument of eq. 4; here f(t, .) is read between the samples by a periodic Catmull-Rom
 * cubic (reading R23, after SPEC.md:147-159):
 *   flat_samples [S][n_knots][N_d] device: f(t, q / n_knots), q = 0..n_knots-1 (mask positions in
 *   periods, R3); n_knots >= 4 (EI_ERR_SHAPE otherwise).
 *   s_mod = exp(-R[h]) f(t, m - m_o(theta) - z gamma dR[h]/dt)   (no centre parameter: the
 *   measured curve carries it)
 * Everything else exactly as ei_forward_h / ei_cost_grad_h. */
int ei_forward_hs(const ei_plan *plan, const float *h, float gamma, const float *flat_samples,
                  int n_knots, const float *mask_pos, const float *drift, float *s_mod, void *stream);
int ei_cost_grad_hs(const ei_plan *plan, const float *h, float gamma, const float *flat_samples,
                    int n_knots, const float *mask_pos, const float *drift, const float *s_exp,
                    float lambda, double *cost, float *g_h, float *g_drift, int32_t *status,
                    void *stream);

/* ei_cost_grad with HOST buffers (same shapes and meaning; status is overwritten, not
 * accumulated).  Copies inputs host->device, evaluates, copies cost, gradients and status
 * back, and returns when they are complete.  The work is ordered after everything already
 * queued on `stream` and runs on the plan's own streams: the maps/flat/mask/drift upload first,
 * the s_exp upload (the bulk of the bytes) on a copy stream overlapping K0/K1 (K2 waits for it).
 * With pinned host memory the whole call is captured once into a CUDA graph and replayed while
 * the 13 pointers and lambda stay the same and every host buffer is still page-locked (checked
 * with cudaPointerGetAttributes on each call; one launch instead of ~20 API calls; env
 * EI_HOST_GRAPH=0 disables; pageable memory, or arguments whose capture failed, take direct
 * calls).  Stacks (>= 8 slices)
 * run in chunks of slices (4 / 8 / 16 chunks from 8 / 16 / 32 slices; env EI_HOST_CHUNKS=K, up to
 * 32, 1 disables), each evaluated by an internal sub-plan of the same geometry, so chunk c's
 * upload, chunk c-1's evaluation and the downloads of earlier chunks overlap (C4: 34.5 ms in one
 * piece, 25.1 ms in 8 chunks, 23.7 ms in 16); chunking is used only when
 * the sub-plans compute bit-identical results (no K3 angle split, same K1 row split).  Device
 * staging buffers, sub-plans, streams, events and the graph belong to the plan (created by the
 * first call, kept until ei_plan_destroy; EI_ERR_RESOURCE if that fails). */
int ei_cost_grad_host(ei_plan *plan, const float *mu, const float *delta, const float *sigma,
                      const float *flat, const float *mask_pos, const float *drift,
                      const float *s_exp, float lambda, double *cost, float *g_mu, float *g_delta,
                      float *g_sigma, int32_t *status, void *stream);

/* Launch accounting (the "one projection + one adjoint per map per evaluation" contract):
 * out[0] = K1 launches, out[1] = maps projected, out[2] = K3 launches, out[3] = maps
 * back-projected, out[4] = K2 launches, out[5] = all libei kernel launches, since plan
 * creation.  Host counters; no device synchronisation. */
int ei_plan_stats(const ei_plan *plan, int64_t out[6]);

/* Per-kernel device timing of ei_cost_grad (measurement support, bench.py).
 * ei_plan_set_timing(plan, max_evals): from now on the next `max_evals` ei_cost_grad(_drift/_h) calls
 * record CUDA events around each of their kernels on the call's stream (max_evals = 0
 * disables; events are created here, EI_ERR_RESOURCE on failure).
 * ei_plan_read_timing(plan, ms[6], n_evals): synchronises the recorded events and returns the
 * summed milliseconds of [K0 pack (+input check), K1 project, K2 curve (+fused K4 cost),
 * K3 backproject, 0, 0] over the recorded calls and their number; then resets the recording. */
int ei_plan_set_timing(ei_plan *plan, int max_evals);
int ei_plan_read_timing(ei_plan *plan, double ms[6], int *n_evals);

/* Launch-plan diagnostics (synchronous: reads a device counter).  out[0] = K1 angle groups,
 * out[1] = K1 rows per staged chunk, out[2] = K1 window-width bound (entries), out[3] = K1 row
 * split of the cost path, out[4] = staged-window overflows seen so far (must be 0: K1 checks the
 * first and last row of every staged chunk, where its taps are extreme; -DEI_CHECK builds also
 * check every K3 tap),
 * out[5] = K1 dynamic shared memory per CTA (bytes), out[6] = K1 angle groups using the
 * ray-fastest lane mapping, out[7] = K3 angle split (most parts of one tile), out[8] = mirror angle pairs (theta,
 * theta + pi) of a 360-degree scan projected and back-projected once (env EI_MIRROR=0 at plan
 * creation disables), out[9] = K2 detector segments per row, out[10] = K1B band mode: map rows
 * per band of the cost / forward path (0: ray-tile units; then out[3] is the number of bands),
 * out[11] = CTAs of the cost path's K1 grid.  The caller's array holds 12 entries. */
int ei_plan_info(const ei_plan *plan, int64_t out[12]);

/* Human-readable name of an EI_* code (static string). */
const char *ei_error_string(int code);

/* Library build identifier, e.g. "libei sm_100a <git-describe>". */
const char *ei_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EI_H */
