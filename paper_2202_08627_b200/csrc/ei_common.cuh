// ei_common.cuh — plan layout and kernel-launcher declarations shared by the libei sources.
// Product code only (never includes or links anything under oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ei.h"

namespace ei {

// Per-angle tables built on the host in fp64 and stored as fp32 (plan.cu, reading R5):
//   k1[a] = {ic, tn, scale, rowdom}   projector (K1), dominant-axis frame:
//           x*(k,i) = (k-(Nd-1)/2)*ic - tn*(i-(N-1)/2) + (N-1)/2,   ic = du/(c_dom*dx),
//           tn = s_oth/c_dom, scale = dx/|c_dom|; rowdom = 1 -> sample rows of the map,
//           0 -> sample rows of the transposed map (= columns) with (cos,sin) swapped.
//   k3[a] = {cdu, sdu, inv_h, scale}  adjoint (K3): k* = x_j*cdu + y_i*sdu + (Nd-1)/2,
//           cdu = cos*dx/du, sdu = sin*dx/du (pixel-index units), inv_h = du/(|c_dom|*dx).
struct Tables {
  float4 *k1 = nullptr;
  float4 *k3 = nullptr;
};

}  // namespace ei

struct ei_plan {
  ei_geometry g{};
  int S = 0, N = 0, NA = 0, ND = 0, M = 0;
  ei::Tables tab;
  // workspace (allocated in ei_plan_create only)
  float4 *maps4 = nullptr;    // [S][N][N]   (mu, delta, sigma, 0)
  float4 *maps4T = nullptr;   // [S][N][N]   transposed copy (column-dominant angles, H2)
  float *mapT1 = nullptr;     // [S][N][N]   transposed single map (ei_project n_maps=1)
  float4 *sino4 = nullptr;    // [S][NA][ND] packed sinogram (ei_backproject n_maps=3)
  float *P = nullptr;         // [S][3][NA][ND] projections
  float4 *G4 = nullptr;       // [S][NA][ND]  (g_mu, g_delta, g_sigma, 0)
  double *part_curve = nullptr;  // [S][NA] per-row cost partials (K2)
  double *part_reg = nullptr;    // [S][RB] per-tile sum x^2 partials (K0)
  int RB = 0;
  // host-I/O staging (ei_cost_grad_host), allocated on first use
  float *h_maps = nullptr, *h_flat = nullptr, *h_mask = nullptr, *h_drift = nullptr,
        *h_sexp = nullptr, *h_grad = nullptr;
  double *h_cost = nullptr;
  int32_t *h_status = nullptr;
  // launch accounting
  mutable int64_t stats[6] = {0, 0, 0, 0, 0, 0};
  // optional per-kernel timing of ei_cost_grad: 7 events per recorded evaluation
  cudaEvent_t *tev = nullptr;
  int tcap = 0;
  mutable int tn = 0;
};

namespace ei {
// K0 (k_pack.cu)
cudaError_t launch_pack3(const ei_plan &p, const float *mu, const float *delta, const float *sigma,
                         size_t in_stride, bool want_reg, int32_t *status, cudaStream_t st);
cudaError_t launch_transpose1(const ei_plan &p, const float *map, cudaStream_t st);
cudaError_t launch_pack_sino3(const ei_plan &p, const float *sino, cudaStream_t st);
cudaError_t launch_check_small(const ei_plan &p, const float *flat, const float *mask,
                               const float *drift, int32_t *status, cudaStream_t st);
// K1 (k_project.cu)
cudaError_t launch_project3(const ei_plan &p, float *P, cudaStream_t st);
cudaError_t launch_project1(const ei_plan &p, const float *map, float *P, cudaStream_t st);
// K2 / K4 (k_curve.cu)
cudaError_t launch_curve_forward(const ei_plan &p, const float *flat, const float *mask,
                                 const float *drift, float *s_mod, cudaStream_t st);
cudaError_t launch_curve_cost_grad(const ei_plan &p, const float *flat, const float *mask,
                                   const float *drift, const float *s_exp, int32_t *status,
                                   cudaStream_t st);
cudaError_t launch_finalize(const ei_plan &p, float lambda, double *cost, cudaStream_t st);
// K3 (k_backproject.cu)
cudaError_t launch_backproject3(const ei_plan &p, const float4 *G, const float *mu,
                                const float *delta, const float *sigma, float lambda, float *g_mu,
                                float *g_delta, float *g_sigma, size_t out_stride, cudaStream_t st);
cudaError_t launch_backproject1(const ei_plan &p, const float *sino, float *map, cudaStream_t st);
}  // namespace ei
