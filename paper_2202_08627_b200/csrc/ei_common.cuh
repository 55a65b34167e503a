// ei_common.cuh — plan layout and kernel-launcher declarations shared by the libei sources.
// Product code only (never includes or links anything under oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

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

// K1 launch plan (k_project.cu: plan_projector)
struct ProjPlan {
  int2 *groups = nullptr;   // device: {first sorted position, count | ray_fast << 16} per group
  int *order = nullptr;     // device: sorted position -> angle index (row-dominant first)
  int *partner = nullptr;   // device [NA]: the angle theta + pi of a projected angle, or -1
  int n_groups = 0;
  int RT = 64;              // rays per K1 CTA (64, or 32 for small single-wave grids)
  int nsl = 4;              // angle slots per K1 thread (angles per CTA = 4 nsl)
  int k0_early = 0;         // K0 triggers K1's launch at its start (K1 grid smaller than the SMs)
  int nst = 4;              // K1 ring stages
  int E = 0;                // K1 ring-stage capacity (entries; rows x stride of a chunk <= E)
  int ray_fast = 0;         // number of angle groups using the ray-fastest consumer lane mapping
  int rcmax = 0;            // most rows of a chunk (diagnostics)
  int wmax = 0;             // widest chunk window (entries)
  int RS = 1;               // row split of the cost path (partial P summed by K2)
  int4 *chunks1 = nullptr;  // device chunk tables {first entry - 1, W, first row, rows}, RS = 1,
  int *coff1 = nullptr;     //   CSR offsets per unit (group, tile)
  int4 *chunksRS = nullptr; // the same for the row-split cost path, units (rs, group, tile)
  int *coffRS = nullptr;
  int nchmax1 = 0, nchmaxRS = 0;   // most chunks of one unit
  int n_tiles = 0;          // ray tiles per angle group
  int *unit1 = nullptr;     // device: CTA -> work unit (tile, group, slice) for RS = 1 (launch order)
  int *unitRS = nullptr;    // device: the same for the row-split cost path
  int PAD = 0;              // zero entries before/after every pair-layout map row
  int Rp = 0;               // padded row length (entries): N + 1 + 2 PAD, even
  int band = 0;             // K1B band mode for the RS launches (small maps): RS = bands of BR rows
  int BR = 0;               // map rows per band
  int bstride = 0;          // staged row stride of a band (entries, even, >= N + 4)
};

// K2 launch plan (k_curve.cu: plan_curve)
struct CurvePlan {
  int nseg = 1;   // segments per detector row
  int W = 0;      // core positions per segment
  int NT = 0;     // threads per CTA (>= W + 4, multiple of 32)
  int nw = 0;     // warps per CTA (per-warp cost / drift partials per item)
  int ctas = 0;   // persistent grid size
};

}  // namespace ei

// arguments of an ei_cost_grad_host call (the captured graph is valid for exactly these)
struct HostKey {
  const void *p[13];
  float lambda;
  HostKey() : p{}, lambda(0.f) {}
  HostKey(const void *a, const void *b, const void *c, const void *d, const void *e, const void *f,
          const void *g, float lam, const void *h, const void *i, const void *j, const void *k,
          const void *l)
      : p{a, b, c, d, e, f, g, h, i, j, k, l, nullptr}, lambda(lam) {}
  bool operator==(const HostKey &o) const {
    for (int q = 0; q < 13; ++q)
      if (p[q] != o.p[q]) return false;
    return lambda == o.lambda;
  }
};

struct ei_plan {
  ei_geometry g{};
  int S = 0, N = 0, NA = 0, ND = 0, M = 0;
  ei::Tables tab;
  ei::ProjPlan proj;
  ei::CurvePlan k2;
  // workspace (allocated in ei_plan_create only)
  // maps in the PAIR layout (k_pack.cu): entry e = (x[e-1], x[e]), e = 0..N, stored at e + PAD
  // in rows of proj.Rp entries (zero padding both sides); *T = the transposed maps (H2)
  float4 *MA = nullptr, *MAT = nullptr;   // [S][N][Rp] (mu0, mu1, delta0, delta1)
  float2 *MB = nullptr, *MBT = nullptr;   // [S][N][Rp] (sigma0, sigma1)
  float2 *M1 = nullptr, *M1T = nullptr;   // [S][N][Rp] single map (ei_project n_maps=1)
  float *P = nullptr;         // [RS][S][3][NA][ND] (partial) projections
  int32_t *diag = nullptr;    // device counter of internal window overflows (must stay 0)
  // gradient sinograms read by K3, stored at entry e + PADG in rows of RpG entries (RpG a multiple
  // of 4; zero padding both sides, written once at plan creation), zero outside the detector:
  //  * three maps, TRIPLE layout, e = -1..ND: GA = (m[e-1], m[e], s[e-1], s[e]),
  //    GB = (d[e-1], d[e], m[e+1], d[e+1]), GC = s[e+1]  (m, d, s: mu, delta, sigma gradients)
  //  * single map, PAIR layout, e = 0..ND: GA1 = (g[e-1], g[e])
  float4 *GA = nullptr;       // [S][NA][RpG]
  float4 *GB = nullptr;       // [S][NA][RpG]
  float *GC = nullptr;        // [S][NA][RpG]
  float2 *GA1 = nullptr;      // [S][NA][RpG]
  int PADG = 0, RpG = 0;
  double *part_curve = nullptr;  // [S][NA][nseg][nw] per-warp cost partials (K2, fp64)
  float *part_mo = nullptr;      // [S][NA][nseg][nw] per-warp dS/dm_o partials (K2, NEXT-2)
  double *part_reg = nullptr;    // [S][RB] per-tile sum x^2 partials (K0)
  float *part3 = nullptr;        // [KS][S][3][N][N] K3 angle-split partial gradients
  int KS = 1;                    // K3 angle split: most parts of one (slice, tile)
  int KSk = 1, KSe = 0;          // (slice, tile) pairs v < KSe have KSk + 1 parts, the rest KSk
  int4 *k3u = nullptr;           // device [n_k3u] K3 units {tile, slice, part, parts} in launch order
  int n_k3u = 0;                 // (only for split grids with more units than SMs)

  // 360-degree scans: angle pairs (theta, theta + pi) sample the same lines (mirrored detector,
  // R6), so K1 projects only the primary angle of each pair and writes both rows, and K3 back-
  // projects only primaries after the gradient rows are folded: G(a) += mirror(G(partner))
  int npairs = 0;                // number of (primary, mirror) pairs
  int NA3 = 0;                   // angles K3 back-projects (primaries + unpaired)
  int *alist3 = nullptr;         // device [NA3] their indices
  int2 *pairs = nullptr;         // device [npairs] (primary, mirror)
  int RB = 0;
  // host-I/O staging (ei_cost_grad_host), allocated on first use
  float *h_maps = nullptr, *h_flat = nullptr, *h_mask = nullptr, *h_drift = nullptr,
        *h_sexp = nullptr, *h_grad = nullptr;
  double *h_cost = nullptr;
  int32_t *h_status = nullptr;
  cudaStream_t h_copy = nullptr;            // s_exp upload stream (host path)
  cudaStream_t h_work = nullptr;            // host path work stream (graph capture / replay)
  cudaEvent_t h_ev[4] = {nullptr, nullptr, nullptr, nullptr};   // small inputs up / s_exp up /
                                                                // caller order / call done
  cudaGraphExec_t h_exec = nullptr;         // captured host path, replayed for the same arguments
  HostKey h_key{};
  int64_t h_stats[6] = {0, 0, 0, 0, 0, 0};  // launch accounting of one captured call
  HostKey h_fail_key{};         // arguments whose graph capture failed (direct path for them)
  bool h_graph_failed = false;  // h_fail_key is set
  // stacks: the host path runs in chunks of slices (sub-plans of h_Sc and of the last chunk's
  // slice count) so uploads, evaluation and downloads of different chunks overlap
  std::vector<double> angles;               // host copy (sub-plan creation)
  int h_nchunk = 0, h_Sc = 0;               // 0: not decided yet, 1: one piece
  ei_plan *h_sub[2] = {nullptr, nullptr};
  cudaStream_t h_down = nullptr;            // download stream (chunked host path)
  static constexpr int HCHUNK_MAX = 32;
  cudaEvent_t h_cev[2 * HCHUNK_MAX + 1] = {};   // per chunk: uploaded, evaluated; + downloads done
  // launch accounting
  mutable int64_t stats[6] = {0, 0, 0, 0, 0, 0};
  // optional per-kernel timing of ei_cost_grad: 7 events per recorded evaluation
  cudaEvent_t *tev = nullptr;
  int tcap = 0;
  mutable int tn = 0;
};

namespace ei {
// launch `kern` on `st` with programmatic stream serialization (PDL): the kernel's prologue may
// overlap the predecessor's tail; the kernel itself calls pdl_wait() before reading its inputs
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, ((KArgs)args)...);
}

int plan_projector(ei_plan &p, const double *angles, const std::vector<int> &proj_angles,
                   std::vector<int2> &groups, std::vector<int> &order, std::vector<int4> &chunks1,
                   std::vector<int> &coff1, std::vector<int4> &chunksRS, std::vector<int> &coffRS,
                   std::vector<int> &unit1, std::vector<int> &unitRS);
size_t k1_smem(int nst, int E, int nchmax, int nmap);   // K1 dynamic shared memory (bytes)
size_t k1_band_smem(int BR, int stride, int nmap);      // K1B (band mode) dynamic shared memory
// fold of mirror-pair gradient rows (k_pack.cu): G(primary) += mirror(G(mirror)), pair layout
cudaError_t launch_fold(const ei_plan &p, int n_maps, cudaStream_t st);
// K0 (k_pack.cu)
struct SmallCheck {          // flat/mask/drift non-finite scan folded into K0
  const float *flat = nullptr, *mask = nullptr, *drift = nullptr;
  int nflat_per_slice = 0;   // flat elements per slice (0: 3 N_d, the Gaussian parameters)
};
cudaError_t launch_pack3(const ei_plan &p, const float *mu, const float *delta, const float *sigma,
                         size_t in_stride, bool want_reg, int32_t *status, SmallCheck chk,
                         cudaStream_t st);
cudaError_t launch_pack1(const ei_plan &p, const float *map, cudaStream_t st, bool want_reg = false,
                         int32_t *status = nullptr, SmallCheck chk = SmallCheck{});
int reg_blocks(int N);
cudaError_t launch_pack_sino(const ei_plan &p, const float *sino, int n_maps, cudaStream_t st);
// K1 (k_project.cu)
cudaError_t launch_project3(const ei_plan &p, float *P, int RS, cudaStream_t st);
cudaError_t launch_project1(const ei_plan &p, float *P, cudaStream_t st, int RS = 1);
// K2 (k_curve.cu)
int plan_curve(ei_plan &p);
cudaError_t launch_curve_forward(const ei_plan &p, const float *flat, const float *mask,
                                 const float *drift, float *s_mod, cudaStream_t st);
cudaError_t launch_curve_cost_grad(const ei_plan &p, const float *flat, const float *mask,
                                   const float *drift, const float *s_exp, int32_t *status,
                                   cudaStream_t st);
cudaError_t launch_curve_forward_h(const ei_plan &p, float gamma, const float *flat, const float *mask,
                                   const float *drift, float *s_mod, cudaStream_t st);
cudaError_t launch_curve_cost_grad_h(const ei_plan &p, float gamma, const float *flat,
                                     const float *mask, const float *drift, const float *s_exp,
                                     int32_t *status, cudaStream_t st);
cudaError_t launch_curve_forward_hs(const ei_plan &p, float gamma, const float *fs, int n_knots,
                                    const float *mask, const float *drift, float *s_mod, cudaStream_t st);
cudaError_t launch_curve_cost_grad_hs(const ei_plan &p, float gamma, const float *fs, int n_knots,
                                      const float *mask, const float *drift, const float *s_exp,
                                      int32_t *status, cudaStream_t st);
// K3 (k_backproject.cu); with `fin` set, the CTAs (0, 0, s) also run the fused K4 finalize:
// cost[s] = fixed-order sum of K2's per-segment partials + lambda * K0's sum x^2 partials, and
// g_drift[s][theta] = sum of K2's per-segment dS/dm_o partials (if g_drift != NULL)
struct Finalize {
  double *cost = nullptr;
  float *g_drift = nullptr;
};
cudaError_t launch_backproject3(const ei_plan &p, const float *mu, const float *delta,
                                const float *sigma, float lambda, float *g_mu, float *g_delta,
                                float *g_sigma, size_t out_stride, const Finalize *fin,
                                cudaStream_t st);
cudaError_t launch_backproject1(const ei_plan &p, float *map, cudaStream_t st, const float *h = nullptr,
                                float lambda = 0.f, const Finalize *fin = nullptr);
int bp_tiles(int N);
int bp_pad();
int bp_chunks(int NA);
}  // namespace ei
