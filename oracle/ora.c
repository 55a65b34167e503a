/*
 * oracle/ora.c — fp64 CPU oracle for the edge-illumination (EI) cost+gradient hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2202_08627_b200/csrc) and the
 * product never links it.
 *
 * What it computes (citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * R# = reading listed in DESIGN.md §3, frozen from SURVEY.md §8(c)):
 *
 *   P_x   = R_J[x]                    Joseph ray-driven projection, eq. 1, R5-R8
 *   Delta = z * D P_delta             refraction shift, eq. 2; D = finite
 *                                     differences along t, R9
 *   T     = exp(-clamp(P_mu,-50,50))  attenuation, eq. 2; clamp per S:308 (R12)
 *   W^2   = max(w^2 + P_sigma, w^2/100)   scattering broadening (R1, R13)
 *   u     = m - c - m_o(theta) - Delta    eq. 4 with m_r == 0, R10, R14
 *   s_mod = T * A * (w/W) * exp(-u^2/(2 W^2))   flat Gaussian IC (R2) convolved with N(0,W^2-w^2)
 *   S     = sum_{theta,t,m} (s_mod - s_exp)^2 + lambda * sum x^2     eq. 5, R11
 *   grad  = R_J^T [dS/dP_x]          analytic chain rule; R_J^T is the literal
 *                                     transpose of the projection loops (ray-driven scatter)
 *
 * Plain loops, fp64 accumulators, deterministic summation order; OpenMP only over
 * independent outputs (angles for the projection, image rows/columns for the scatter),
 * so results do not depend on the thread count.
 *
 * Parity pins: see tests/test_oracle_*.py.  The scattering term (R1) has no paper value:
 * beyond the self-consistency pins (limits, Gaussian-convolution quadrature, moments,
 * finite differences) it is "parity unpinned" against the paper.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------
 * a1: Joseph projection of one N x N map (row-major, x = column index j contiguous)
 *     onto one sinogram [n_angles][n_det].  SURVEY.md §8(a) a1; R5-R8, R22.
 *     Pixel centres x_j = (j-(N-1)/2)*dx, y_i = (i-(N-1)/2)*dx; detector u_k = (k-(Nd-1)/2)*du;
 *     ray: x cos(theta) + y sin(theta) = u_k.
 * ------------------------------------------------------------------------------- */
static int row_dominant(double c, double s) { return fabs(c) >= fabs(s); }

void ora_project(int n, int n_angles, int n_det, double dx, double du, const double *angles,
                 const double *img, double *sino)
{
    const double ctr = 0.5 * (n - 1), dctr = 0.5 * (n_det - 1);
#pragma omp parallel for schedule(dynamic, 1)
    for (int a = 0; a < n_angles; ++a) {
        const double c = cos(angles[a]), s = sin(angles[a]);
        for (int k = 0; k < n_det; ++k) {
            const double u = (k - dctr) * du;
            double acc = 0.0;
            if (row_dominant(c, s)) {
                for (int i = 0; i < n; ++i) {                       /* one sample per row */
                    const double y = (i - ctr) * dx;
                    const double xs = ((u - y * s) / c) / dx + ctr;
                    const double f = floor(xs);
                    const int j0 = (int)f;
                    const double w = xs - f;
                    if (j0 >= 0 && j0 < n) acc += (1.0 - w) * img[(size_t)i * n + j0];
                    if (j0 + 1 >= 0 && j0 + 1 < n) acc += w * img[(size_t)i * n + j0 + 1];
                }
                acc *= dx / fabs(c);
            } else {
                for (int j = 0; j < n; ++j) {                       /* one sample per column */
                    const double x = (j - ctr) * dx;
                    const double ys = ((u - x * c) / s) / dx + ctr;
                    const double f = floor(ys);
                    const int i0 = (int)f;
                    const double w = ys - f;
                    if (i0 >= 0 && i0 < n) acc += (1.0 - w) * img[(size_t)i0 * n + j];
                    if (i0 + 1 >= 0 && i0 + 1 < n) acc += w * img[(size_t)(i0 + 1) * n + j];
                }
                acc *= dx / fabs(s);
            }
            sino[(size_t)a * n_det + k] = acc;
        }
    }
}

/* ---------------------------------------------------------------------------------
 * a5 (oracle form): R_J^T as a ray-driven SCATTER — the same loops as ora_project with
 * every gather "acc += w * img[p]" replaced by "img[p] += w * g".  S:58-61 (adjoint =
 * exact transpose).  To stay thread-count independent without atomics the loops are
 * run in two passes: row-dominant angles parallel over image rows i (a row-dominant
 * ray touches row i only at its row-i sample), column-dominant angles parallel over
 * columns j.  Within a pixel, contributions are added in (angle, ray) ascending order.
 * ------------------------------------------------------------------------------- */
void ora_backproject(int n, int n_angles, int n_det, double dx, double du, const double *angles,
                     const double *sino, double *img)
{
    const double ctr = 0.5 * (n - 1), dctr = 0.5 * (n_det - 1);
    memset(img, 0, sizeof(double) * (size_t)n * n);
#pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < n; ++i) {
        const double y = (i - ctr) * dx;
        for (int a = 0; a < n_angles; ++a) {
            const double c = cos(angles[a]), s = sin(angles[a]);
            if (!row_dominant(c, s)) continue;
            const double scale = dx / fabs(c);
            for (int k = 0; k < n_det; ++k) {
                const double g = sino[(size_t)a * n_det + k] * scale;
                const double u = (k - dctr) * du;
                const double xs = ((u - y * s) / c) / dx + ctr;
                const double f = floor(xs);
                const int j0 = (int)f;
                const double w = xs - f;
                if (j0 >= 0 && j0 < n) img[(size_t)i * n + j0] += (1.0 - w) * g;
                if (j0 + 1 >= 0 && j0 + 1 < n) img[(size_t)i * n + j0 + 1] += w * g;
            }
        }
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int j = 0; j < n; ++j) {
        const double x = (j - ctr) * dx;
        for (int a = 0; a < n_angles; ++a) {
            const double c = cos(angles[a]), s = sin(angles[a]);
            if (row_dominant(c, s)) continue;
            const double scale = dx / fabs(s);
            for (int k = 0; k < n_det; ++k) {
                const double g = sino[(size_t)a * n_det + k] * scale;
                const double u = (k - dctr) * du;
                const double ys = ((u - x * c) / s) / dx + ctr;
                const double f = floor(ys);
                const int i0 = (int)f;
                const double w = ys - f;
                if (i0 >= 0 && i0 < n) img[(size_t)i0 * n + j] += (1.0 - w) * g;
                if (i0 + 1 >= 0 && i0 + 1 < n) img[(size_t)(i0 + 1) * n + j] += w * g;
            }
        }
    }
}

/* ---------------------------------------------------------------------------------
 * a2: D along t ("finite differences"): central inside, one-sided at the
 * two ends, divided by du.  Requires n_det >= 3.
 * ------------------------------------------------------------------------------- */
void ora_diff_t(int n_det, double du, const double *p, double *d)
{
    d[0] = (p[1] - p[0]) / du;
    for (int k = 1; k < n_det - 1; ++k) d[k] = (p[k + 1] - p[k - 1]) / (2.0 * du);
    d[n_det - 1] = (p[n_det - 1] - p[n_det - 2]) / du;
}

/* D^T written out explicitly: row k of D scatters its coefficients times g[k]. */
void ora_diff_t_adjoint(int n_det, double du, const double *g, double *y)
{
    for (int j = 0; j < n_det; ++j) y[j] = 0.0;
    y[0] += -g[0] / du;
    y[1] += g[0] / du;
    for (int k = 1; k < n_det - 1; ++k) {
        y[k - 1] += -g[k] / (2.0 * du);
        y[k + 1] += g[k] / (2.0 * du);
    }
    y[n_det - 2] += -g[n_det - 1] / du;
    y[n_det - 1] += g[n_det - 1] / du;
}

/* ---------------------------------------------------------------------------------
 * a2-a4 for one detector row (one slice, one angle): the curve model, residual, cost
 * and dS/dP.  SURVEY.md §8(a) a2-a4; eq. 2, eq. 4, eq. 5.
 *
 *   p_mu, p_delta, p_sigma : [n_det] projections of this row
 *   flat_A, flat_c, flat_w : [n_det] Gaussian flat-IC parameters (R2)
 *   mask                   : [n_mask] mask positions (R3)
 *   drift                  : m_o(theta) of this row (R14)
 *   s_exp                  : [n_mask][n_det] measured curves, or NULL (forward only)
 *   s_mod                  : [n_mask][n_det] output, or NULL
 *   cost                   : += sum r^2 (only when s_exp != NULL)
 *   g_mu, g_delta, g_sigma : [n_det] dS/dP_x (only when s_exp != NULL); g_delta already
 *                            includes z * D^T
 *   counters[0..1]         : += mu-clamp hits, W^2-clamp hits (R12, R13)
 *   g_drift                : += dS/dm_o(theta) of this row, or NULL (NEXT-2: m_o enters eq. 4,
 *                            P:74-75, through u = m - c - m_o - Delta, so ds/dm_o = s u / W^2)
 * ------------------------------------------------------------------------------- */
void ora_curve_row(int n_det, int n_mask, double du, double z,
                   const double *p_mu, const double *p_delta, const double *p_sigma,
                   const double *flat_A, const double *flat_c, const double *flat_w,
                   const double *mask, double drift, const double *s_exp, double *s_mod,
                   double *cost, double *g_mu, double *g_delta, double *g_sigma,
                   int64_t *counters, double *g_drift)
{
    double *dP = (double *)malloc(sizeof(double) * n_det);
    double *gD = (double *)malloc(sizeof(double) * n_det);
    ora_diff_t(n_det, du, p_delta, dP);
    double S = 0.0, Gmo = 0.0;
    for (int k = 0; k < n_det; ++k) {
        const double delta_shift = z * dP[k];                          /* Delta = z dR[delta]/dt */
        double pm = p_mu[k];
        int mu_clamped = 0;
        if (pm > 50.0) { pm = 50.0; mu_clamped = 1; }
        if (pm < -50.0) { pm = -50.0; mu_clamped = 1; }
        const double T = exp(-pm);
        const double w = flat_w[k];
        double W2 = w * w + p_sigma[k];
        int w2_clamped = 0;
        if (W2 < w * w / 100.0) { W2 = w * w / 100.0; w2_clamped = 1; }
        counters[0] += mu_clamped;
        counters[1] += w2_clamped;
        const double W = sqrt(W2);
        double gm = 0.0, gd = 0.0, gs = 0.0;
        for (int m = 0; m < n_mask; ++m) {
            const double u = mask[m] - flat_c[k] - drift - delta_shift;
            const double s = T * flat_A[k] * (w / W) * exp(-u * u / (2.0 * W2));
            if (s_mod) s_mod[(size_t)m * n_det + k] = s;
            if (s_exp) {
                const double r = s - s_exp[(size_t)m * n_det + k];
                S += r * r;
                gm += -2.0 * r * s;                                   /* ds/dP_mu = -s        */
                gd += 2.0 * r * s * u / W2;                           /* ds/dDelta = s u/W^2  */
                gs += r * s * (u * u - W2) / (W2 * W2);               /* 2 r ds/dW^2          */
                Gmo += 2.0 * r * s * u / W2;                          /* ds/dm_o = s u/W^2    */
            }
        }
        if (s_exp) {
            g_mu[k] = mu_clamped ? 0.0 : gm;
            gD[k] = gd;
            g_sigma[k] = w2_clamped ? 0.0 : gs;
        }
    }
    if (s_exp) {
        ora_diff_t_adjoint(n_det, du, gD, g_delta);                   /* g_delta = z D^T g_Delta */
        for (int k = 0; k < n_det; ++k) g_delta[k] *= z;
        *cost += S;
        if (g_drift) *g_drift += Gmo;
    }
    free(dP);
    free(gD);
}

static int64_t count_nonfinite(const float *p, size_t n)
{
    int64_t c = 0;
    for (size_t i = 0; i < n; ++i) c += !isfinite(p[i]);
    return c;
}

/* ---------------------------------------------------------------------------------
 * Whole-slice forward model (S:206 'forward'): maps -> s_mod [n_angles][n_mask][n_det].
 * Inputs are the fp32 arrays the GPU reads, widened to fp64 here.
 * ------------------------------------------------------------------------------- */
static double *widen(const float *p, size_t n)
{
    double *d = (double *)malloc(sizeof(double) * n);
    for (size_t i = 0; i < n; ++i) d[i] = (double)p[i];
    return d;
}

static void project3(int n, int n_angles, int n_det, double dx, double du, const double *angles,
                     const float *mu, const float *delta, const float *sigma,
                     double *Pm, double *Pd, double *Ps)
{
    const size_t nn = (size_t)n * n;
    double *m = widen(mu, nn), *d = widen(delta, nn), *s = widen(sigma, nn);
    ora_project(n, n_angles, n_det, dx, du, angles, m, Pm);
    ora_project(n, n_angles, n_det, dx, du, angles, d, Pd);
    ora_project(n, n_angles, n_det, dx, du, angles, s, Ps);
    free(m); free(d); free(s);
}

void ora_forward(int n, int n_angles, int n_det, int n_mask, double dx, double du, double z,
                 const double *angles, const float *mu, const float *delta, const float *sigma,
                 const float *flat /*[3][n_det]*/, const float *mask, const float *drift /*or NULL*/,
                 double *s_mod /*[n_angles][n_mask][n_det]*/, int64_t *counters /*[2]*/)
{
    const size_t ns = (size_t)n_angles * n_det;
    double *Pm = malloc(sizeof(double) * ns), *Pd = malloc(sizeof(double) * ns),
           *Ps = malloc(sizeof(double) * ns);
    project3(n, n_angles, n_det, dx, du, angles, mu, delta, sigma, Pm, Pd, Ps);
    double *fl = widen(flat, (size_t)3 * n_det), *mk = widen(mask, n_mask);
    int64_t cnt[2] = {0, 0};
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : cnt[:2])
    for (int a = 0; a < n_angles; ++a) {
        int64_t c2[2] = {0, 0};
        ora_curve_row(n_det, n_mask, du, z, Pm + (size_t)a * n_det, Pd + (size_t)a * n_det,
                      Ps + (size_t)a * n_det, fl, fl + n_det, fl + 2 * n_det, mk,
                      drift ? (double)drift[a] : 0.0, NULL, s_mod + (size_t)a * n_mask * n_det,
                      NULL, NULL, NULL, NULL, c2, NULL);
        cnt[0] += c2[0];
        cnt[1] += c2[1];
    }
    counters[0] += cnt[0];
    counters[1] += cnt[1];
    free(Pm); free(Pd); free(Ps); free(fl); free(mk);
}

/* ---------------------------------------------------------------------------------
 * Whole-slice cost and gradient (S:261 'cost' + S:270 'grad', map blocks only).
 *   status[0] += non-finite input elements (maps, flat, mask, drift, s_exp)
 *   status[1] += mu-clamp hits, status[2] += W^2-clamp hits
 *   g_drift   = [n_angles] dS/dm_o(theta) of this slice (NEXT-2), or NULL
 * ------------------------------------------------------------------------------- */
void ora_cost_grad2(int n, int n_angles, int n_det, int n_mask, double dx, double du, double z,
                    const double *angles, const float *mu, const float *delta, const float *sigma,
                    const float *flat, const float *mask, const float *drift, const float *s_exp,
                    double lambda, double *cost, double *g_mu, double *g_delta, double *g_sigma,
                    int64_t *status /*[3]*/, double *g_drift)
{
    const size_t nn = (size_t)n * n, ns = (size_t)n_angles * n_det;
    status[0] += count_nonfinite(mu, nn) + count_nonfinite(delta, nn) + count_nonfinite(sigma, nn) +
                 count_nonfinite(flat, (size_t)3 * n_det) + count_nonfinite(mask, n_mask) +
                 (drift ? count_nonfinite(drift, n_angles) : 0) +
                 count_nonfinite(s_exp, ns * n_mask);
    double *Pm = malloc(sizeof(double) * ns), *Pd = malloc(sizeof(double) * ns),
           *Ps = malloc(sizeof(double) * ns);
    double *Gm = malloc(sizeof(double) * ns), *Gd = malloc(sizeof(double) * ns),
           *Gs = malloc(sizeof(double) * ns);
    double *rowcost = calloc(n_angles, sizeof(double));
    project3(n, n_angles, n_det, dx, du, angles, mu, delta, sigma, Pm, Pd, Ps);
    double *fl = widen(flat, (size_t)3 * n_det), *mk = widen(mask, n_mask);
    int64_t cnt[2] = {0, 0};
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : cnt[:2])
    for (int a = 0; a < n_angles; ++a) {
        int64_t c2[2] = {0, 0};
        double *se = widen(s_exp + (size_t)a * n_mask * n_det, (size_t)n_mask * n_det);
        ora_curve_row(n_det, n_mask, du, z, Pm + (size_t)a * n_det, Pd + (size_t)a * n_det,
                      Ps + (size_t)a * n_det, fl, fl + n_det, fl + 2 * n_det, mk,
                      drift ? (double)drift[a] : 0.0, se, NULL, &rowcost[a],
                      Gm + (size_t)a * n_det, Gd + (size_t)a * n_det, Gs + (size_t)a * n_det, c2,
                      g_drift ? &g_drift[a] : NULL);
        free(se);
        cnt[0] += c2[0];
        cnt[1] += c2[1];
    }
    status[1] += cnt[0];
    status[2] += cnt[1];
    double S = 0.0;
    for (int a = 0; a < n_angles; ++a) S += rowcost[a];               /* fixed angle order */
    ora_backproject(n, n_angles, n_det, dx, du, angles, Gm, g_mu);
    ora_backproject(n, n_angles, n_det, dx, du, angles, Gd, g_delta);
    ora_backproject(n, n_angles, n_det, dx, du, angles, Gs, g_sigma);
    if (lambda > 0.0) {                                               /* eq. 5 regulariser (R11) */
        double reg = 0.0;
        for (size_t p = 0; p < nn; ++p) {
            reg += (double)mu[p] * mu[p] + (double)delta[p] * delta[p] + (double)sigma[p] * sigma[p];
            g_mu[p] += 2.0 * lambda * mu[p];
            g_delta[p] += 2.0 * lambda * delta[p];
            g_sigma[p] += 2.0 * lambda * sigma[p];
        }
        S += lambda * reg;
    }
    *cost = S;
    free(Pm); free(Pd); free(Ps); free(Gm); free(Gd); free(Gs); free(rowcost); free(fl); free(mk);
}

void ora_cost_grad(int n, int n_angles, int n_det, int n_mask, double dx, double du, double z,
                   const double *angles, const float *mu, const float *delta, const float *sigma,
                   const float *flat, const float *mask, const float *drift, const float *s_exp,
                   double lambda, double *cost, double *g_mu, double *g_delta, double *g_sigma,
                   int64_t *status /*[3]*/)
{
    ora_cost_grad2(n, n_angles, n_det, n_mask, dx, du, z, angles, mu, delta, sigma, flat, mask, drift,
                   s_exp, lambda, cost, g_mu, g_delta, g_sigma, status, NULL);
}

/* ---------------------------------------------------------------------------------
 * NEXT-3: the paper's own single-map model, eq. 4 with m_r == 0, under the
 * homogeneity assumption mu = gamma^-1 delta = h, cost eq. 5 with the L2 term on h:
 *
 *   P     = R_J[h]
 *   T     = exp(-clamp(P, -50, 50))                      (R12)
 *   u     = m - c - m_o(theta) - z gamma D P             (eq. 4; R10 sign)
 *   s_mod = T * f(t, u + c) = T * A * exp(-u^2 / (2 w^2))   (Gaussian flat IC, R2; no scattering)
 *   S     = sum (s_mod - s_exp)^2 + lambda sum h^2
 *   dS/dP = -2 sum_m r s  [0 where clamped]  +  z gamma D^T ( 2 sum_m r s u / w^2 )
 *   grad  = R_J^T dS/dP + 2 lambda h
 *
 * Written out directly from eq. 4 (its own loops, not via the three-map functions above).
 * flat [3][n_det] = (A, c, w); s_exp [n_angles][n_mask][n_det]; grad [n][n]; s_mod (or NULL)
 * [n_angles][n_mask][n_det]; status[0] += non-finite inputs, status[1] += clamp hits.
 * ------------------------------------------------------------------------------- */
void ora_cost_grad_h(int n, int n_angles, int n_det, int n_mask, double dx, double du, double z,
                     double gamma, const double *angles, const float *h, const float *flat,
                     const float *mask, const float *drift, const float *s_exp, double lambda,
                     double *cost, double *grad, double *s_mod, int64_t *status)
{
    const size_t nn = (size_t)n * n, ns = (size_t)n_angles * n_det;
    if (s_exp)
        status[0] += count_nonfinite(h, nn) + count_nonfinite(flat, (size_t)3 * n_det) +
                     count_nonfinite(mask, n_mask) + (drift ? count_nonfinite(drift, n_angles) : 0) +
                     count_nonfinite(s_exp, ns * n_mask);
    double *hd = widen(h, nn);
    double *P = malloc(sizeof(double) * ns), *G = malloc(sizeof(double) * ns);
    double *rowcost = calloc(n_angles, sizeof(double));
    ora_project(n, n_angles, n_det, dx, du, angles, hd, P);
    int64_t clamps = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : clamps)
    for (int a = 0; a < n_angles; ++a) {
        const double *Pa = P + (size_t)a * n_det;
        double *dP = malloc(sizeof(double) * n_det), *gD = malloc(sizeof(double) * n_det),
               *gT = malloc(sizeof(double) * n_det), *y = malloc(sizeof(double) * n_det);
        ora_diff_t(n_det, du, Pa, dP);
        const double mo = drift ? (double)drift[a] : 0.0;
        double Sa = 0.0;
        for (int k = 0; k < n_det; ++k) {
            double pk = Pa[k];
            int cl = 0;
            if (pk > 50.0) { pk = 50.0; cl = 1; }
            if (pk < -50.0) { pk = -50.0; cl = 1; }
            clamps += cl;
            const double T = exp(-pk);
            const double A = flat[k], c = flat[n_det + k], w = flat[2 * n_det + k];
            double g_t = 0.0, g_d = 0.0;
            for (int m = 0; m < n_mask; ++m) {
                const double u = (double)mask[m] - c - mo - z * gamma * dP[k];
                const double s = T * A * exp(-u * u / (2.0 * w * w));
                if (s_mod) s_mod[((size_t)a * n_mask + m) * n_det + k] = s;
                if (s_exp) {
                    const double r = s - (double)s_exp[((size_t)a * n_mask + m) * n_det + k];
                    Sa += r * r;
                    g_t += -2.0 * r * s;                    /* d/dP through T: ds/dP = -s   */
                    g_d += 2.0 * r * s * u / (w * w);       /* d/dShift: ds/dShift = s u/w^2 */
                }
            }
            gT[k] = cl ? 0.0 : g_t;
            gD[k] = g_d;
        }
        if (s_exp) {
            ora_diff_t_adjoint(n_det, du, gD, y);        /* shift = z gamma D P */
            for (int k = 0; k < n_det; ++k) G[(size_t)a * n_det + k] = gT[k] + z * gamma * y[k];
            rowcost[a] = Sa;
        }
        free(dP); free(gD); free(gT); free(y);
    }
    if (s_exp) {
        status[1] += clamps;
        double S = 0.0;
        for (int a = 0; a < n_angles; ++a) S += rowcost[a];
        ora_backproject(n, n_angles, n_det, dx, du, angles, G, grad);
        if (lambda > 0.0) {
            double reg = 0.0;
            for (size_t q = 0; q < nn; ++q) {
                reg += hd[q] * hd[q];
                grad[q] += 2.0 * lambda * hd[q];
            }
            S += lambda * reg;
        }
        *cost = S;
    }
    free(hd); free(P); free(G); free(rowcost);
}

/* ---------------------------------------------------------------------------------
 * NEXT-4: the measured (sampled) flat-field IC.  The paper measures f(t, m) by scanning the
 * sample mask over one period in 33 steps, repeated 20 times; f at the shifted argument
 * of eq. 4 is read between the samples.  The paper does not say how (SPEC.md's reading,
 * S:147-159, adopted here as reading R23): a PERIODIC Catmull-Rom cubic through the K knots
 * m_q = q / K (mask positions in periods, R3, period 1):
 *   x = m K, i = floor(x), tau = x - i, p_j = f[(i - 1 + j) mod K], j = 0..3
 *   f(m)  = 1/2 [2 p1 + (p2 - p0) tau + (2 p0 - 5 p1 + 4 p2 - p3) tau^2 + (3 p1 - p0 - 3 p2 + p3) tau^3]
 *   f'(m) = K/2 [(p2 - p0) + 2 (2 p0 - 5 p1 + 4 p2 - p3) tau + 3 (3 p1 - p0 - 3 p2 + p3) tau^2]
 * fs: [n_knots][n_det] samples (t contiguous).
 * ------------------------------------------------------------------------------- */
void ora_ic_eval(const float *fs, int n_knots, int n_det, int t, double m, double *f, double *fp)
{
    const double x = m * n_knots;
    const double fl = floor(x);
    const double tau = x - fl;
    long long i = (long long)fl;
    double p[4];
    for (int j = 0; j < 4; ++j) {
        long long q = (i - 1 + j) % n_knots;
        if (q < 0) q += n_knots;
        p[j] = (double)fs[(size_t)q * n_det + t];
    }
    const double a1 = p[2] - p[0];
    const double a2 = 2.0 * p[0] - 5.0 * p[1] + 4.0 * p[2] - p[3];
    const double a3 = 3.0 * p[1] - p[0] - 3.0 * p[2] + p[3];
    *f = 0.5 * (2.0 * p[1] + a1 * tau + a2 * tau * tau + a3 * tau * tau * tau);
    *fp = 0.5 * n_knots * (a1 + 2.0 * a2 * tau + 3.0 * a3 * tau * tau);
}

/* The single-map model (eq. 4) with the sampled flat IC: as ora_cost_grad_h but
 *   s_mod = T f(t, m - m_o - z gamma D P),   ds/dShift = -T f'(t, .)
 *   dS/dP = -2 sum_m r s [0 where clamped] + z gamma D^T (-2 sum_m r T f') */
void ora_cost_grad_hs(int n, int n_angles, int n_det, int n_mask, int n_knots, double dx, double du,
                      double z, double gamma, const double *angles, const float *h, const float *fs,
                      const float *mask, const float *drift, const float *s_exp, double lambda,
                      double *cost, double *grad, double *s_mod, int64_t *status)
{
    const size_t nn = (size_t)n * n, ns = (size_t)n_angles * n_det;
    if (s_exp)
        status[0] += count_nonfinite(h, nn) + count_nonfinite(fs, (size_t)n_knots * n_det) +
                     count_nonfinite(mask, n_mask) + (drift ? count_nonfinite(drift, n_angles) : 0) +
                     count_nonfinite(s_exp, ns * n_mask);
    double *hd = widen(h, nn);
    double *P = malloc(sizeof(double) * ns), *G = malloc(sizeof(double) * ns);
    double *rowcost = calloc(n_angles, sizeof(double));
    ora_project(n, n_angles, n_det, dx, du, angles, hd, P);
    int64_t clamps = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : clamps)
    for (int a = 0; a < n_angles; ++a) {
        const double *Pa = P + (size_t)a * n_det;
        double *dP = malloc(sizeof(double) * n_det), *gD = malloc(sizeof(double) * n_det),
               *gT = malloc(sizeof(double) * n_det), *y = malloc(sizeof(double) * n_det);
        ora_diff_t(n_det, du, Pa, dP);
        const double mo = drift ? (double)drift[a] : 0.0;
        double Sa = 0.0;
        for (int k = 0; k < n_det; ++k) {
            double pk = Pa[k];
            int cl = 0;
            if (pk > 50.0) { pk = 50.0; cl = 1; }
            if (pk < -50.0) { pk = -50.0; cl = 1; }
            clamps += cl;
            const double T = exp(-pk);
            double g_t = 0.0, g_d = 0.0;
            for (int m = 0; m < n_mask; ++m) {
                double f, fp;
                ora_ic_eval(fs, n_knots, n_det, k, (double)mask[m] - mo - z * gamma * dP[k], &f, &fp);
                const double s = T * f;
                if (s_mod) s_mod[((size_t)a * n_mask + m) * n_det + k] = s;
                if (s_exp) {
                    const double r = s - (double)s_exp[((size_t)a * n_mask + m) * n_det + k];
                    Sa += r * r;
                    g_t += -2.0 * r * s;                    /* d/dP through T               */
                    g_d += -2.0 * r * T * fp;               /* d/dShift: ds/dShift = -T f'  */
                }
            }
            gT[k] = cl ? 0.0 : g_t;
            gD[k] = g_d;
        }
        if (s_exp) {
            ora_diff_t_adjoint(n_det, du, gD, y);
            for (int k = 0; k < n_det; ++k) G[(size_t)a * n_det + k] = gT[k] + z * gamma * y[k];
            rowcost[a] = Sa;
        }
        free(dP); free(gD); free(gT); free(y);
    }
    if (s_exp) {
        status[1] += clamps;
        double S = 0.0;
        for (int a = 0; a < n_angles; ++a) S += rowcost[a];
        ora_backproject(n, n_angles, n_det, dx, du, angles, G, grad);
        if (lambda > 0.0) {
            double reg = 0.0;
            for (size_t q = 0; q < nn; ++q) {
                reg += hd[q] * hd[q];
                grad[q] += 2.0 * lambda * hd[q];
            }
            S += lambda * reg;
        }
        *cost = S;
    }
    free(hd); free(P); free(G); free(rowcost);
}

int ora_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
