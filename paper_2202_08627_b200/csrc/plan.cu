// plan.cu — the C ABI of libei (include/ei.h): argument validation, plan/workspace
// management and the launch sequence of each entry point.  Host code only; the kernels
// live in k_*.cu.  No CPU fallback exists: every numeric step runs in the kernels.
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <utility>
#include <new>
#include <vector>

#include "ei_common.cuh"

#ifndef EI_GIT_DESCRIBE
#define EI_GIT_DESCRIBE "dev"
#endif

namespace {

int check_geom(const ei_geometry *g) {
  if (!g) return EI_ERR_NULL;
  if (g->n_slices < 1 || g->n < 2 || g->n_angles < 1 || g->n_det < 3 || g->n_mask < 1)
    return EI_ERR_SHAPE;
  // sizes must fit the 32-bit per-slice index arithmetic of the kernels
  if ((int64_t)g->n * g->n > (1LL << 30) || (int64_t)g->n_angles * g->n_det * g->n_mask > (1LL << 30))
    return EI_ERR_RESOURCE;
  // size limits of this implementation: 16 N_d + 4 M <= 220 KB and N_theta <= 14080 (parity is
  // tested at both limits, tests/test_gpu_limits.py; BASELINE's configurations use 3072 and 1440); K2's staging ring bounds M separately
  // (plan_curve: the projections + M measured rows of a segment must fit a CTA's shared memory)
  if (16LL * g->n_det + 4LL * g->n_mask > 220 * 1024 || 16LL * g->n_angles > 220 * 1024)
    return EI_ERR_SHAPE;
  if (!(isfinite(g->pixel) && isfinite(g->det_pitch) && isfinite(g->z))) return EI_ERR_DOMAIN;
  if (g->pixel <= 0 || g->det_pitch <= 0 || g->z <= 0) return EI_ERR_DOMAIN;
  if (g->det_pitch < g->pixel) return EI_ERR_DOMAIN;   // <= 2 taps in the adjoint (a5)
  return EI_OK;
}

template <class T>
cudaError_t dalloc(T **p, size_t count) {
  return cudaMalloc((void **)p, count * sizeof(T) + 16);
}

void free_timing(ei_plan *p) {
  if (p->tev) {
    for (int i = 0; i < 7 * p->tcap; ++i) cudaEventDestroy(p->tev[i]);   // 5 used per eval
    delete[] p->tev;
  }
  p->tev = nullptr;
  p->tcap = 0;
  p->tn = 0;
}

void free_plan(ei_plan *p) {
  if (!p) return;
  free_timing(p);
  if (p->h_exec) cudaGraphExecDestroy(p->h_exec);
  for (ei_plan *q : p->h_sub)
    if (q) free_plan(q);
  for (cudaEvent_t ev : p->h_cev)
    if (ev) cudaEventDestroy(ev);
  for (cudaStream_t q : {p->h_copy, p->h_work, p->h_down})
    if (q) {
      cudaStreamSynchronize(q);
      cudaStreamDestroy(q);
    }
  for (cudaEvent_t ev : p->h_ev)
    if (ev) cudaEventDestroy(ev);
  void *ptrs[] = {p->tab.k1, p->tab.k3, p->proj.groups, p->proj.order, p->proj.partner, p->alist3,
                  p->pairs, p->proj.chunks1, p->proj.coff1, p->proj.chunksRS, p->proj.coffRS, p->proj.unit1, p->proj.unitRS, p->MA, p->MAT, p->MB,
                  p->MBT, p->M1, p->M1T, p->diag, p->part_mo, p->part3, p->k3u, p->P, p->GA, p->GB, p->GC, p->GA1,
                  p->part_curve, p->part_reg, p->h_maps, p->h_flat, p->h_mask, p->h_drift,
                  p->h_sexp, p->h_grad, p->h_cost, p->h_status};
  for (void *q : ptrs)
    if (q) cudaFree(q);
  delete p;
}

inline int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? EI_OK : EI_ERR_CUDA;
}

}  // namespace

extern "C" {

const char *ei_error_string(int code) {
  switch (code) {
    case EI_OK: return "ok";
    case EI_ERR_NULL: return "null pointer argument";
    case EI_ERR_SHAPE: return "invalid shape";
    case EI_ERR_DOMAIN: return "argument out of domain";
    case EI_ERR_RESOURCE: return "device resource allocation failed";
    case EI_ERR_CUDA: return "CUDA error";
    default: return "unknown error code";
  }
}

const char *ei_version(void) { return "libei sm_100a " EI_GIT_DESCRIBE; }

int ei_plan_create(const ei_geometry *geom, const double *angles, ei_plan **out) {
  if (!out) return EI_ERR_NULL;
  *out = nullptr;
  int rc = check_geom(geom);
  if (rc) return rc;
  if (!angles) return EI_ERR_NULL;
  for (int a = 0; a < geom->n_angles; ++a)
    if (!isfinite(angles[a])) return EI_ERR_DOMAIN;

  ei_plan *p = new (std::nothrow) ei_plan();
  if (!p) return EI_ERR_RESOURCE;
  p->g = *geom;
  p->S = geom->n_slices;
  p->N = geom->n;
  p->NA = geom->n_angles;
  p->ND = geom->n_det;
  p->M = geom->n_mask;
  p->angles.assign(angles, angles + geom->n_angles);
  const double dx = geom->pixel, du = geom->det_pitch;

  // a0: per-angle tables in fp64 -> fp32 (reading R5: row-dominant iff
  // |cos| >= |sin| evaluated in fp64)
  const int NA = p->NA;
  float4 *k1 = new float4[NA], *k3 = new float4[NA];
  for (int a = 0; a < NA; ++a) {
    const double c = cos(angles[a]), s = sin(angles[a]);
    const bool rowdom = fabs(c) >= fabs(s);
    const double cd = rowdom ? c : s, so = rowdom ? s : c;
    k1[a] = make_float4((float)(du / (cd * dx)), (float)(so / cd), (float)(dx / fabs(cd)),
                        rowdom ? 1.f : 0.f);
    k3[a] = make_float4((float)(c * dx / du), (float)(s * dx / du), (float)(du / (fabs(cd) * dx)),
                        (float)(dx / fabs(cd)));
  }
  // mirror pairs of 360-degree scans: theta and theta + pi (mod 2 pi, to 1e-9 rad) sample the same
  // lines with the detector mirrored (R6), so only the primary (angle mod 2 pi < pi) is projected
  // and back-projected (tuning knob EI_MIRROR=0 switches this off)
  std::vector<int> partner(NA, -1), prim;
  std::vector<int2> pairs;
  {
    const char *env = getenv("EI_MIRROR");
    if (!env || atoi(env) != 0) {
      auto wrap = [](double t) { t = fmod(t, 2 * M_PI); return t < 0 ? t + 2 * M_PI : t; };
      std::vector<std::pair<double, int>> w(NA);
      for (int a = 0; a < NA; ++a) w[a] = {wrap(angles[a]), a};
      std::sort(w.begin(), w.end());
      std::vector<char> used(NA, 0);
      for (int q = 0; q < NA; ++q) {
        const double ta = w[q].first;
        const int a = w[q].second;
        if (ta >= M_PI || used[a]) continue;
        auto it = std::lower_bound(w.begin(), w.end(), std::make_pair(ta + M_PI - 1e-9, -1));
        for (; it != w.end() && it->first <= ta + M_PI + 1e-9; ++it) {
          const int b = it->second;
          if (b != a && !used[b]) {
            partner[a] = b;
            used[a] = used[b] = 1;
            pairs.push_back(make_int2(a, b));
            break;
          }
        }
      }
    }
    std::vector<char> is_mirror(NA, 0);
    for (const int2 &q : pairs) is_mirror[q.y] = 1;
    for (int a = 0; a < NA; ++a)
      if (!is_mirror[a]) prim.push_back(a);
  }
  p->npairs = (int)pairs.size();
  p->NA3 = (int)prim.size();
  std::vector<int2> groups;
  std::vector<int4> chunks1, chunksRS;
  std::vector<int> order, unit1, unitRS, coff1, coffRS;
  rc = ei::plan_projector(*p, angles, prim, groups, order, chunks1, coff1, chunksRS, coffRS, unit1, unitRS);
  if (!rc) rc = ei::plan_curve(*p);
  if (rc) {
    delete[] k1;
    delete[] k3;
    delete p;
    return rc;
  }
  const size_t S = p->S, SINO = (size_t)p->NA * p->ND;
  const size_t NP = (size_t)p->N * p->proj.Rp;
  p->RB = ei::reg_blocks(p->N);
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  A(dalloc(&p->tab.k1, NA));
  A(dalloc(&p->tab.k3, NA));
  A(dalloc(&p->proj.groups, groups.size()));
  A(dalloc(&p->proj.order, order.size()));
  A(dalloc(&p->proj.partner, NA));
  A(dalloc(&p->alist3, prim.size()));
  if (!pairs.empty()) A(dalloc(&p->pairs, pairs.size()));
  A(dalloc(&p->proj.chunks1, std::max<size_t>(1, chunks1.size())));
  A(dalloc(&p->proj.coff1, coff1.size()));
  if (!coffRS.empty()) {
    A(dalloc(&p->proj.chunksRS, std::max<size_t>(1, chunksRS.size())));
    A(dalloc(&p->proj.coffRS, coffRS.size()));
  }
  A(dalloc(&p->proj.unit1, unit1.size()));
  A(dalloc(&p->proj.unitRS, unitRS.size()));
  A(dalloc(&p->MA, S * NP));
  A(dalloc(&p->MAT, S * NP));
  A(dalloc(&p->MB, S * NP));
  A(dalloc(&p->MBT, S * NP));
  A(dalloc(&p->M1, S * NP));
  A(dalloc(&p->M1T, S * NP));
  A(dalloc(&p->diag, 1));
  p->PADG = ei::bp_pad();
  p->RpG = (p->ND + 2 + 2 * p->PADG + 3) & ~3;   // multiple of 4: 16-B aligned C-plane rows
  const size_t SINO1 = (size_t)p->NA * p->RpG;
  A(dalloc(&p->P, (size_t)p->proj.RS * S * 3 * SINO));
  A(dalloc(&p->GA, S * SINO1));
  A(dalloc(&p->GB, S * SINO1));
  A(dalloc(&p->GC, S * SINO1));
  A(dalloc(&p->GA1, S * SINO1));
  A(dalloc(&p->part_curve, S * NA * p->k2.nseg * p->k2.nw));
  A(dalloc(&p->part_mo, S * NA * p->k2.nseg * p->k2.nw));
  A(dalloc(&p->part_reg, S * p->RB));
  // K3 angle split for small grids: the largest KS (<= 16, <= angle chunks) keeping the grid within
  // one wave of 3 CTAs per SM; the KS partial gradients are summed by ks_reduce_kernel (measured:
  // C1 KS 1 -> 6-8: 22.5 -> 14.5 us; C2 KS 4-6 best)
  // The first `extra` (slice, tile) pairs take one part more, so the grid fills the 3 x SMs slots
  // exactly (C2: 60 tiles in 7 parts and 4 in 6 = 444 CTAs instead of 64 x 6 = 384; the 6-part
  // units placed heaviest first on the least-loaded SM): C2 K3 33.8 -> 31.8 us.
  std::vector<int4> k3u;
  {
    int sms = 148, dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaGetLastError();
    const int T = ei::bp_tiles(p->N), C = ei::bp_chunks(p->NA3);
    const long long ctas = (long long)T * p->S, slots = 3LL * sms;
    int KS = 1;
    while (KS < 16 && KS + 1 <= C && ctas * (KS + 1) <= slots) ++KS;
    long long extra = (KS < 16 && KS + 1 <= C && ctas * KS < slots) ? std::min(ctas, slots - ctas * KS) : 0;
    if (const char *e = getenv("EI_K3_KS")) {   // tuning knob: uniform split
      KS = std::max(1, std::min(16, atoi(e)));
      extra = 0;
    }
    if (ctas * KS + extra <= sms) extra = 0;   // tiny grid: uniform split, block-index decode
    p->KSk = KS;
    p->KSe = (int)extra;
    p->KS = KS + (extra > 0 ? 1 : 0);
    const long long n = ctas * KS + extra;
    if (p->KS > 1 && n > sms) {   // placement table: parts heaviest first, least-loaded SM
      std::vector<int4> u;
      for (int s = 0; s < p->S; ++s)
        for (int t = 0; t < T; ++t) {
          const int np = KS + ((long long)s * T + t < extra ? 1 : 0);
          for (int q = 0; q < np; ++q) u.push_back(make_int4(t, s, q, np));
        }
      std::vector<int> ord(u.size());
      for (size_t i = 0; i < u.size(); ++i) ord[i] = (int)i;
      std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return u[a].w < u[b].w; });
      std::vector<int> cap(sms, 0), used(sms, 0);
      std::vector<double> load(sms, 0.0);
      for (size_t b = 0; b < u.size(); ++b) cap[b % sms] += 1;
      k3u.assign(u.size(), make_int4(0, 0, 0, 1));
      for (int i : ord) {
        int best = -1;
        for (int m = 0; m < sms; ++m)
          if (used[m] < cap[m] && (best < 0 || load[m] < load[best])) best = m;
        k3u[best + used[best] * sms] = u[i];
        used[best] += 1;
        load[best] += 1.0 / u[i].w;   // the part's share of the angles
      }
      p->n_k3u = (int)u.size();
      A(dalloc(&p->k3u, k3u.size()));
    }
  }
  if (p->KS > 1) A(dalloc(&p->part3, (size_t)p->KS * S * 3 * p->N * p->N));
  if (e == cudaSuccess) A(cudaMemcpy(p->tab.k1, k1, sizeof(float4) * NA, cudaMemcpyHostToDevice));
  if (e == cudaSuccess) A(cudaMemcpy(p->tab.k3, k3, sizeof(float4) * NA, cudaMemcpyHostToDevice));
  if (e == cudaSuccess)
    A(cudaMemcpy(p->proj.groups, groups.data(), sizeof(int2) * groups.size(), cudaMemcpyHostToDevice));
  if (e == cudaSuccess)
    A(cudaMemcpy(p->proj.order, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice));
  if (e == cudaSuccess)
    A(cudaMemcpy(p->proj.partner, partner.data(), sizeof(int) * NA, cudaMemcpyHostToDevice));
  {   // K3's angle list: cos >= 0 first (the pixel-pair roles of the three-map adjoint flip with
      // the sign of cos, k_backproject.cu), each class in angle-index order
    std::vector<int> al(prim);
    std::stable_sort(al.begin(), al.end(), [&](int x, int y) { return (cos(angles[x]) < 0) < (cos(angles[y]) < 0); });
    if (e == cudaSuccess) A(cudaMemcpy(p->alist3, al.data(), sizeof(int) * al.size(), cudaMemcpyHostToDevice));
  }
  if (e == cudaSuccess && !pairs.empty())
    A(cudaMemcpy(p->pairs, pairs.data(), sizeof(int2) * pairs.size(), cudaMemcpyHostToDevice));
  if (e == cudaSuccess) A(cudaMemset(p->diag, 0, sizeof(int32_t)));
  if (e == cudaSuccess && p->k3u)
    A(cudaMemcpy(p->k3u, k3u.data(), sizeof(int4) * k3u.size(), cudaMemcpyHostToDevice));

  // the zero padding of the map rows is written once here; K0 only writes the interior
  for (void *q : {(void *)p->MA, (void *)p->MAT})
    if (e == cudaSuccess) A(cudaMemset(q, 0, sizeof(float4) * S * NP));
  for (void *q : {(void *)p->MB, (void *)p->MBT, (void *)p->M1, (void *)p->M1T})
    if (e == cudaSuccess) A(cudaMemset(q, 0, sizeof(float2) * S * NP));
  if (e == cudaSuccess) A(cudaMemset(p->GA, 0, sizeof(float4) * S * SINO1));   // zero padding
  if (e == cudaSuccess) A(cudaMemset(p->GB, 0, sizeof(float4) * S * SINO1));
  if (e == cudaSuccess) A(cudaMemset(p->GC, 0, sizeof(float) * S * SINO1));
  if (e == cudaSuccess) A(cudaMemset(p->GA1, 0, sizeof(float2) * S * SINO1));
  if (e == cudaSuccess && !chunks1.empty())
    A(cudaMemcpy(p->proj.chunks1, chunks1.data(), sizeof(int4) * chunks1.size(), cudaMemcpyHostToDevice));
  if (e == cudaSuccess) A(cudaMemcpy(p->proj.coff1, coff1.data(), sizeof(int) * coff1.size(), cudaMemcpyHostToDevice));
  if (e == cudaSuccess && !coffRS.empty()) {
    if (!chunksRS.empty())
      A(cudaMemcpy(p->proj.chunksRS, chunksRS.data(), sizeof(int4) * chunksRS.size(), cudaMemcpyHostToDevice));
    A(cudaMemcpy(p->proj.coffRS, coffRS.data(), sizeof(int) * coffRS.size(), cudaMemcpyHostToDevice));
  }
  if (e == cudaSuccess)
    A(cudaMemcpy(p->proj.unit1, unit1.data(), sizeof(int) * unit1.size(), cudaMemcpyHostToDevice));
  if (e == cudaSuccess)
    A(cudaMemcpy(p->proj.unitRS, unitRS.data(), sizeof(int) * unitRS.size(), cudaMemcpyHostToDevice));
  delete[] k1;
  delete[] k3;
  if (e != cudaSuccess) {
    cudaGetLastError();
    free_plan(p);
    return e == cudaErrorMemoryAllocation ? EI_ERR_RESOURCE : EI_ERR_CUDA;
  }
  *out = p;
  return EI_OK;
}

void ei_plan_destroy(ei_plan *plan) { free_plan(plan); }

int ei_plan_stats(const ei_plan *p, int64_t out[6]) {
  if (!p || !out) return EI_ERR_NULL;
  for (int i = 0; i < 6; ++i) out[i] = p->stats[i];
  return EI_OK;
}

int ei_plan_info(const ei_plan *p, int64_t out[12]) {
  if (!p || !out) return EI_ERR_NULL;
  int32_t d = 0;
  if (cudaMemcpy(&d, p->diag, sizeof(d), cudaMemcpyDeviceToHost) != cudaSuccess) return EI_ERR_CUDA;
  out[0] = p->proj.n_groups;
  out[1] = p->proj.rcmax;
  out[2] = p->proj.wmax;
  out[3] = p->proj.RS;
  out[4] = d;
  out[5] = (int64_t)ei::k1_smem(p->proj.nst, p->proj.E, std::max(p->proj.nchmax1, p->proj.nchmaxRS), 3);
  out[6] = p->proj.ray_fast;
  out[7] = p->KS;
  out[8] = p->npairs;
  out[9] = p->k2.nseg;
  out[10] = p->proj.band ? p->proj.BR : 0;
  out[11] = p->proj.band ? (int64_t)p->proj.n_groups * p->proj.RS * p->S
                         : (int64_t)p->proj.n_tiles * p->proj.n_groups * p->S * p->proj.RS;
  return EI_OK;
}

int ei_plan_set_timing(ei_plan *p, int max_evals) {
  if (!p) return EI_ERR_NULL;
  if (max_evals < 0) return EI_ERR_DOMAIN;
  free_timing(p);
  if (max_evals == 0) return EI_OK;
  p->tev = new (std::nothrow) cudaEvent_t[7 * (size_t)max_evals];
  if (!p->tev) return EI_ERR_RESOURCE;
  for (int i = 0; i < 7 * max_evals; ++i) {
    if (cudaEventCreate(&p->tev[i]) != cudaSuccess) {
      for (int k = 0; k < i; ++k) cudaEventDestroy(p->tev[k]);
      delete[] p->tev;
      p->tev = nullptr;
      cudaGetLastError();
      return EI_ERR_RESOURCE;
    }
  }
  p->tcap = max_evals;
  p->tn = 0;
  return EI_OK;
}

int ei_plan_read_timing(ei_plan *p, double ms[6], int *n_evals) {
  if (!p || !ms || !n_evals) return EI_ERR_NULL;
  for (int k = 0; k < 6; ++k) ms[k] = 0.0;
  for (int e = 0; e < p->tn; ++e) {
    cudaEvent_t *ev = p->tev + 7 * e;
    if (cudaEventSynchronize(ev[4]) != cudaSuccess) return EI_ERR_CUDA;
    for (int k = 0; k < 4; ++k) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ev[k], ev[k + 1]) != cudaSuccess) return EI_ERR_CUDA;
      ms[k] += t;
    }
  }
  *n_evals = p->tn;
  p->tn = 0;
  return EI_OK;
}

int ei_project(const ei_plan *p, const float *maps, int n_maps, float *sino, void *stream) {
  if (!p || !maps || !sino) return EI_ERR_NULL;
  if (n_maps != 1 && n_maps != 3) return EI_ERR_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t NN = (size_t)p->N * p->N;
  cudaError_t e;
  if (n_maps == 3) {
    // maps [S][3][N][N]: slice stride 3*NN, plane stride NN
    e = ei::launch_pack3(*p, maps, maps + NN, maps + 2 * NN, 3 * NN, false, nullptr,
                         ei::SmallCheck{}, st);
    if (e == cudaSuccess) e = ei::launch_project3(*p, sino, 1, st);
    p->stats[0] += 1;
    p->stats[1] += 3;
    p->stats[5] += 2;
  } else {
    e = ei::launch_pack1(*p, maps, st);
    if (e == cudaSuccess) e = ei::launch_project1(*p, sino, st);
    p->stats[0] += 1;
    p->stats[1] += 1;
    p->stats[5] += 2;
  }
  return cuda_status(e);
}

int ei_backproject(const ei_plan *p, const float *sino, int n_maps, float *maps, void *stream) {
  if (!p || !maps || !sino) return EI_ERR_NULL;
  if (n_maps != 1 && n_maps != 3) return EI_ERR_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t NN = (size_t)p->N * p->N;
  cudaError_t e;
  if (n_maps == 3) {
    e = ei::launch_pack_sino(*p, sino, 3, st);
    if (e == cudaSuccess) e = ei::launch_fold(*p, 3, st);
    if (e == cudaSuccess)
      e = ei::launch_backproject3(*p, nullptr, nullptr, nullptr, 0.f, maps, maps + NN,
                                  maps + 2 * NN, 3 * NN, nullptr, st);
    p->stats[2] += 1;
    p->stats[3] += 3;
    p->stats[5] += 2 + (p->npairs > 0) + (p->KS > 1);
  } else {
    e = ei::launch_pack_sino(*p, sino, 1, st);
    if (e == cudaSuccess) e = ei::launch_fold(*p, 1, st);
    if (e == cudaSuccess) e = ei::launch_backproject1(*p, maps, st);
    p->stats[2] += 1;
    p->stats[3] += 1;
    p->stats[5] += 2 + (p->npairs > 0) + (p->KS > 1);
  }
  return cuda_status(e);
}

int ei_forward(const ei_plan *p, const float *mu, const float *delta, const float *sigma,
               const float *flat, const float *mask, const float *drift, float *s_mod,
               void *stream) {
  if (!p || !mu || !delta || !sigma || !flat || !mask || !s_mod) return EI_ERR_NULL;
  cudaStream_t st = (cudaStream_t)stream;
  // maps given as three [S][N][N] arrays: plane stride handled by pack3 (slice stride NN)
  cudaError_t e = ei::launch_pack3(*p, mu, delta, sigma, (size_t)p->N * p->N, false, nullptr,
                                   ei::SmallCheck{}, st);
  if (e == cudaSuccess) e = ei::launch_project3(*p, p->P, p->proj.RS, st);
  if (e == cudaSuccess) e = ei::launch_curve_forward(*p, flat, mask, drift, s_mod, st);
  p->stats[0] += 1;
  p->stats[1] += 3;
  p->stats[4] += 1;
  p->stats[5] += 3;
  return cuda_status(e);
}

namespace {
// sexp_ready: if not NULL, an event K2 (the first reader of s_exp) waits for (host path: the
// s_exp upload runs on a copy stream under K0 and K1)
int cost_grad_impl(const ei_plan *p, const float *mu, const float *delta, const float *sigma,
                   const float *flat, const float *mask, const float *drift, const float *s_exp,
                   float lambda, double *cost, float *g_mu, float *g_delta, float *g_sigma,
                   float *g_drift, int32_t *status, void *stream, cudaEvent_t sexp_ready = nullptr,
                   bool check_shared = true) {
  if (!p || !mu || !delta || !sigma || !flat || !mask || !s_exp || !cost || !g_mu || !g_delta ||
      !g_sigma || !status)
    return EI_ERR_NULL;
  if (!(lambda >= 0.f) || !isfinite(lambda)) return EI_ERR_DOMAIN;
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t *ev = (p->tev && p->tn < p->tcap) ? p->tev + 7 * p->tn++ : nullptr;
  auto mark = [&](int k) { if (ev) cudaEventRecord(ev[k], st); };
  const size_t NN = (size_t)p->N * p->N;
  // mask / drift are shared by the slices: a chunked call scans them once
  ei::SmallCheck chk{flat, check_shared ? mask : nullptr, check_shared ? drift : nullptr};
  mark(0);
  cudaError_t e = ei::launch_pack3(*p, mu, delta, sigma, NN, lambda > 0.f, status, chk, st);  // K0
  mark(1);
  if (e == cudaSuccess) e = ei::launch_project3(*p, p->P, p->proj.RS, st);          // K1
  mark(2);
  if (e == cudaSuccess && sexp_ready) e = cudaStreamWaitEvent(st, sexp_ready, 0);
  if (e == cudaSuccess) e = ei::launch_curve_cost_grad(*p, flat, mask, drift, s_exp, status, st);  // K2
  mark(3);
  if (e == cudaSuccess) e = ei::launch_fold(*p, 3, st);                              // mirror pairs
  ei::Finalize fin{cost, g_drift};
  if (e == cudaSuccess) e = ei::launch_backproject3(*p, mu, delta, sigma, lambda, g_mu, g_delta,
                                                    g_sigma, NN, &fin, st);            // K3 + K4
  mark(4);
  p->stats[5] += 4 + (p->npairs > 0) + (p->KS > 1);
  p->stats[0] += 1;
  p->stats[1] += 3;
  p->stats[2] += 1;
  p->stats[3] += 3;
  p->stats[4] += 1;
  return cuda_status(e);
}
}  // namespace

int ei_cost_grad(const ei_plan *p, const float *mu, const float *delta, const float *sigma,
                 const float *flat, const float *mask, const float *drift, const float *s_exp,
                 float lambda, double *cost, float *g_mu, float *g_delta, float *g_sigma,
                 int32_t *status, void *stream) {
  return cost_grad_impl(p, mu, delta, sigma, flat, mask, drift, s_exp, lambda, cost, g_mu, g_delta,
                        g_sigma, nullptr, status, stream);
}

int ei_cost_grad_drift(const ei_plan *p, const float *mu, const float *delta, const float *sigma,
                       const float *flat, const float *mask, const float *drift, const float *s_exp,
                       float lambda, double *cost, float *g_mu, float *g_delta, float *g_sigma,
                       float *g_drift, int32_t *status, void *stream) {
  if (!g_drift) return EI_ERR_NULL;
  return cost_grad_impl(p, mu, delta, sigma, flat, mask, drift, s_exp, lambda, cost, g_mu, g_delta,
                        g_sigma, g_drift, status, stream);
}

int ei_forward_h(const ei_plan *p, const float *h, float gamma, const float *flat, const float *mask,
                 const float *drift, float *s_mod, void *stream) {
  if (!p || !h || !flat || !mask || !s_mod) return EI_ERR_NULL;
  if (!isfinite(gamma)) return EI_ERR_DOMAIN;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = ei::launch_pack1(*p, h, st);                                        // K0
  if (e == cudaSuccess) e = ei::launch_project1(*p, p->P, st, p->proj.RS);           // K1
  if (e == cudaSuccess) e = ei::launch_curve_forward_h(*p, gamma, flat, mask, drift, s_mod, st);  // K2
  p->stats[0] += 1;
  p->stats[1] += 1;
  p->stats[4] += 1;
  p->stats[5] += 3;
  return cuda_status(e);
}

int ei_cost_grad_h(const ei_plan *p, const float *h, float gamma, const float *flat,
                   const float *mask, const float *drift, const float *s_exp, float lambda,
                   double *cost, float *g_h, float *g_drift, int32_t *status, void *stream) {
  if (!p || !h || !flat || !mask || !s_exp || !cost || !g_h || !status) return EI_ERR_NULL;
  if (!(lambda >= 0.f) || !isfinite(lambda) || !isfinite(gamma)) return EI_ERR_DOMAIN;
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t *ev = (p->tev && p->tn < p->tcap) ? p->tev + 7 * p->tn++ : nullptr;
  auto mark = [&](int k) { if (ev) cudaEventRecord(ev[k], st); };
  ei::SmallCheck chk{flat, mask, drift};
  mark(0);
  cudaError_t e = ei::launch_pack1(*p, h, st, lambda > 0.f, status, chk);            // K0
  mark(1);
  if (e == cudaSuccess) e = ei::launch_project1(*p, p->P, st, p->proj.RS);           // K1
  mark(2);
  if (e == cudaSuccess)
    e = ei::launch_curve_cost_grad_h(*p, gamma, flat, mask, drift, s_exp, status, st);  // K2
  mark(3);
  if (e == cudaSuccess) e = ei::launch_fold(*p, 1, st);                              // mirror pairs
  ei::Finalize fin{cost, g_drift};
  if (e == cudaSuccess) e = ei::launch_backproject1(*p, g_h, st, h, lambda, &fin);   // K3 + K4
  mark(4);
  p->stats[0] += 1;
  p->stats[1] += 1;
  p->stats[2] += 1;
  p->stats[3] += 1;
  p->stats[4] += 1;
  p->stats[5] += 4 + (p->npairs > 0) + (p->KS > 1);
  return cuda_status(e);
}

int ei_forward_hs(const ei_plan *p, const float *h, float gamma, const float *flat_samples,
                  int n_knots, const float *mask, const float *drift, float *s_mod, void *stream) {
  if (!p || !h || !flat_samples || !mask || !s_mod) return EI_ERR_NULL;
  if (n_knots < 4) return EI_ERR_SHAPE;
  if (!isfinite(gamma)) return EI_ERR_DOMAIN;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = ei::launch_pack1(*p, h, st);                                        // K0
  if (e == cudaSuccess) e = ei::launch_project1(*p, p->P, st, p->proj.RS);           // K1
  if (e == cudaSuccess)
    e = ei::launch_curve_forward_hs(*p, gamma, flat_samples, n_knots, mask, drift, s_mod, st);  // K2
  p->stats[0] += 1;
  p->stats[1] += 1;
  p->stats[4] += 1;
  p->stats[5] += 3;
  return cuda_status(e);
}

int ei_cost_grad_hs(const ei_plan *p, const float *h, float gamma, const float *flat_samples,
                    int n_knots, const float *mask, const float *drift, const float *s_exp,
                    float lambda, double *cost, float *g_h, float *g_drift, int32_t *status,
                    void *stream) {
  if (!p || !h || !flat_samples || !mask || !s_exp || !cost || !g_h || !status) return EI_ERR_NULL;
  if (n_knots < 4) return EI_ERR_SHAPE;
  if (!(lambda >= 0.f) || !isfinite(lambda) || !isfinite(gamma)) return EI_ERR_DOMAIN;
  cudaStream_t st = (cudaStream_t)stream;
  ei::SmallCheck chk{flat_samples, mask, drift, n_knots * p->ND};
  cudaError_t e = ei::launch_pack1(*p, h, st, lambda > 0.f, status, chk);            // K0
  if (e == cudaSuccess) e = ei::launch_project1(*p, p->P, st, p->proj.RS);           // K1
  if (e == cudaSuccess)
    e = ei::launch_curve_cost_grad_hs(*p, gamma, flat_samples, n_knots, mask, drift, s_exp, status, st);
  if (e == cudaSuccess) e = ei::launch_fold(*p, 1, st);                              // mirror pairs
  ei::Finalize fin{cost, g_drift};
  if (e == cudaSuccess) e = ei::launch_backproject1(*p, g_h, st, h, lambda, &fin);   // K3 + K4
  p->stats[0] += 1;
  p->stats[1] += 1;
  p->stats[2] += 1;
  p->stats[3] += 1;
  p->stats[4] += 1;
  p->stats[5] += 4 + (p->npairs > 0) + (p->KS > 1);
  return cuda_status(e);
}

namespace {
// Chunked host path for stacks (decided on the first host call): K chunks of Sc slices, each
// evaluated by a sub-plan of the same geometry, so chunk c's upload (h_copy), chunk c-1's
// evaluation (st) and chunk c-2's download (h_down) overlap.  Only when the sub-plans compute
// exactly what the whole plan computes: no K3 angle split and the same K1 row split (every other
// planning choice leaves each slice's arithmetic unchanged), so the results are bit-identical.
// Env EI_HOST_CHUNKS=K sets the count (1 disables; default 16 for >= 32 slices, 8 for >= 16, 4 for
// >= 8; C4 e2e per call 8 / 16 / 32 chunks: 25.1 / 23.7 / 24.1 ms, tools/dbg/sweep_chunks.sh).
void setup_chunks(ei_plan *p) {
  p->h_nchunk = 1;
  const char *env = getenv("EI_HOST_CHUNKS");
  int want = env ? atoi(env) : (p->S >= 32 ? 16 : (p->S >= 16 ? 8 : (p->S >= 8 ? 4 : 1)));
  want = std::min(std::min(want, p->S), ei_plan::HCHUNK_MAX);
  if (want <= 1 || p->KS != 1) return;
  const int Sc = (p->S + want - 1) / want, n = (p->S + Sc - 1) / Sc, Sl = p->S - (n - 1) * Sc;
  if (n <= 1) return;
  ei_geometry g = p->g;
  ei_plan *sub[2] = {nullptr, nullptr};
  bool ok = true;
  for (int k = 0; k < 2 && ok; ++k) {
    if (k == 1 && Sl == Sc) break;
    g.n_slices = k == 0 ? Sc : Sl;
    ok = ei_plan_create(&g, p->angles.data(), &sub[k]) == EI_OK && sub[k]->KS == 1 &&
         sub[k]->proj.RS == p->proj.RS && sub[k]->k2.nseg == p->k2.nseg;
  }
  cudaError_t e = cudaSuccess;
  if (ok) e = cudaStreamCreateWithFlags(&p->h_down, cudaStreamNonBlocking);
  for (int k = 0; k < 2 * n + 1 && ok && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&p->h_cev[k], cudaEventDisableTiming);
  if (!ok || e != cudaSuccess) {
    cudaGetLastError();
    for (ei_plan *q : sub)
      if (q) free_plan(q);
    return;   // one piece
  }
  p->h_sub[0] = sub[0];
  p->h_sub[1] = sub[1];
  p->h_Sc = Sc;
  p->h_nchunk = n;
}

int enqueue_host_chunked(ei_plan *p, const float *mu, const float *delta, const float *sigma,
                         const float *flat, const float *mask, const float *drift, const float *s_exp,
                         float lambda, double *cost, float *g_mu, float *g_delta, float *g_sigma,
                         int32_t *status, cudaStream_t st) {
  const size_t S = p->S, NN = (size_t)p->N * p->N, ND = p->ND, NA = p->NA, M = p->M;
  const int n = p->h_nchunk;
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  const cudaMemcpyKind H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost;
  A(cudaMemcpyAsync(p->h_mask, mask, sizeof(float) * M, H2D, st));
  if (drift) A(cudaMemcpyAsync(p->h_drift, drift, sizeof(float) * NA, H2D, st));
  A(cudaMemsetAsync(p->h_status, 0, sizeof(int32_t) * 4, st));
  A(cudaEventRecord(p->h_ev[0], st));
  A(cudaStreamWaitEvent(p->h_copy, p->h_ev[0], 0));
  A(cudaStreamWaitEvent(p->h_down, p->h_ev[0], 0));
  if (e != cudaSuccess) return EI_ERR_CUDA;
  float *dm[3] = {p->h_maps, p->h_maps + S * NN, p->h_maps + 2 * S * NN};
  float *dg[3] = {p->h_grad, p->h_grad + S * NN, p->h_grad + 2 * S * NN};
  const float *hm[3] = {mu, delta, sigma};
  float *hg[3] = {g_mu, g_delta, g_sigma};
  for (int c = 0; c < n; ++c) {
    const size_t s0 = (size_t)c * p->h_Sc, sc = std::min((size_t)p->h_Sc, S - s0);
    ei_plan *q = sc == (size_t)p->h_Sc ? p->h_sub[0] : p->h_sub[1];
    for (int k = 0; k < 3; ++k)
      A(cudaMemcpyAsync(dm[k] + s0 * NN, hm[k] + s0 * NN, sizeof(float) * sc * NN, H2D, p->h_copy));
    A(cudaMemcpyAsync(p->h_flat + s0 * 3 * ND, flat + s0 * 3 * ND, sizeof(float) * sc * 3 * ND, H2D, p->h_copy));
    const size_t se = NA * M * ND;
    A(cudaMemcpyAsync(p->h_sexp + s0 * se, s_exp + s0 * se, sizeof(float) * sc * se, H2D, p->h_copy));
    A(cudaEventRecord(p->h_cev[2 * c], p->h_copy));
    A(cudaStreamWaitEvent(st, p->h_cev[2 * c], 0));
    if (e != cudaSuccess) return EI_ERR_CUDA;
    int64_t s_before[6];
    for (int i = 0; i < 6; ++i) s_before[i] = q->stats[i];
    int rc = cost_grad_impl(q, dm[0] + s0 * NN, dm[1] + s0 * NN, dm[2] + s0 * NN, p->h_flat + s0 * 3 * ND,
                            p->h_mask, drift ? p->h_drift : nullptr, p->h_sexp + s0 * se, lambda,
                            p->h_cost + s0, dg[0] + s0 * NN, dg[1] + s0 * NN, dg[2] + s0 * NN, nullptr,
                            p->h_status, st, nullptr, c == 0);
    for (int i = 0; i < 6; ++i) p->stats[i] += q->stats[i] - s_before[i];
    if (rc) return rc;
    A(cudaEventRecord(p->h_cev[2 * c + 1], st));
    A(cudaStreamWaitEvent(p->h_down, p->h_cev[2 * c + 1], 0));
    A(cudaMemcpyAsync(cost + s0, p->h_cost + s0, sizeof(double) * sc, D2H, p->h_down));
    for (int k = 0; k < 3; ++k)
      A(cudaMemcpyAsync(hg[k] + s0 * NN, dg[k] + s0 * NN, sizeof(float) * sc * NN, D2H, p->h_down));
  }
  A(cudaMemcpyAsync(status, p->h_status, sizeof(int32_t) * 4, D2H, st));
  A(cudaEventRecord(p->h_cev[2 * n], p->h_down));
  A(cudaStreamWaitEvent(st, p->h_cev[2 * n], 0));
  return e == cudaSuccess ? EI_OK : EI_ERR_CUDA;
}

// the host path's device work (uploads, K0..K3, downloads) enqueued on st (+ the copy stream)
int enqueue_host_path(ei_plan *p, const float *mu, const float *delta, const float *sigma,
                      const float *flat, const float *mask, const float *drift, const float *s_exp,
                      float lambda, double *cost, float *g_mu, float *g_delta, float *g_sigma,
                      int32_t *status, cudaStream_t st) {
  const size_t S = p->S, NN = (size_t)p->N * p->N, ND = p->ND, NA = p->NA, M = p->M;
  const size_t nsexp = S * NA * M * ND;
  if (p->h_nchunk > 1)
    return enqueue_host_chunked(p, mu, delta, sigma, flat, mask, drift, s_exp, lambda, cost, g_mu,
                                g_delta, g_sigma, status, st);
  cudaError_t e = cudaSuccess;
  auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  const cudaMemcpyKind H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost;
  // the small inputs first on the compute stream, so K0/K1 start after ~1/6 of the bytes; the
  // s_exp upload (the bulk: M values per ray) follows on the copy stream, overlapping K0 and K1,
  // and K2 waits for it (event h_ev[1])
  float *dmu = p->h_maps, *ddl = p->h_maps + S * NN, *dsg = p->h_maps + 2 * S * NN;
  A(cudaMemcpyAsync(dmu, mu, sizeof(float) * S * NN, H2D, st));
  A(cudaMemcpyAsync(ddl, delta, sizeof(float) * S * NN, H2D, st));
  A(cudaMemcpyAsync(dsg, sigma, sizeof(float) * S * NN, H2D, st));
  A(cudaMemcpyAsync(p->h_flat, flat, sizeof(float) * S * 3 * ND, H2D, st));
  A(cudaMemcpyAsync(p->h_mask, mask, sizeof(float) * M, H2D, st));
  if (drift) A(cudaMemcpyAsync(p->h_drift, drift, sizeof(float) * NA, H2D, st));
  A(cudaMemsetAsync(p->h_status, 0, sizeof(int32_t) * 4, st));
  A(cudaEventRecord(p->h_ev[0], st));
  A(cudaStreamWaitEvent(p->h_copy, p->h_ev[0], 0));
  A(cudaMemcpyAsync(p->h_sexp, s_exp, sizeof(float) * nsexp, H2D, p->h_copy));
  A(cudaEventRecord(p->h_ev[1], p->h_copy));
  if (e != cudaSuccess) return EI_ERR_CUDA;
  float *gm = p->h_grad, *gd = p->h_grad + S * NN, *gs = p->h_grad + 2 * S * NN;
  int rc = cost_grad_impl(p, dmu, ddl, dsg, p->h_flat, p->h_mask, drift ? p->h_drift : nullptr,
                          p->h_sexp, lambda, p->h_cost, gm, gd, gs, nullptr, p->h_status, st,
                          p->h_ev[1]);
  if (rc) return rc;
  A(cudaMemcpyAsync(cost, p->h_cost, sizeof(double) * S, D2H, st));
  A(cudaMemcpyAsync(g_mu, gm, sizeof(float) * S * NN, D2H, st));
  A(cudaMemcpyAsync(g_delta, gd, sizeof(float) * S * NN, D2H, st));
  A(cudaMemcpyAsync(g_sigma, gs, sizeof(float) * S * NN, D2H, st));
  A(cudaMemcpyAsync(status, p->h_status, sizeof(int32_t) * 4, D2H, st));
  return e == cudaSuccess ? EI_OK : EI_ERR_CUDA;
}
}  // namespace

int ei_cost_grad_host(ei_plan *p, const float *mu, const float *delta, const float *sigma,
                      const float *flat, const float *mask, const float *drift,
                      const float *s_exp, float lambda, double *cost, float *g_mu, float *g_delta,
                      float *g_sigma, int32_t *status, void *stream) {
  if (!p || !mu || !delta || !sigma || !flat || !mask || !s_exp || !cost || !g_mu || !g_delta ||
      !g_sigma || !status)
    return EI_ERR_NULL;
  if (!(lambda >= 0.f) || !isfinite(lambda)) return EI_ERR_DOMAIN;
  const size_t S = p->S, NN = (size_t)p->N * p->N, ND = p->ND, NA = p->NA, M = p->M;
  const size_t nsexp = S * NA * M * ND;
  if (!p->h_maps) {
    cudaError_t e = cudaSuccess;
    auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
    A(dalloc(&p->h_maps, 3 * S * NN));
    A(dalloc(&p->h_flat, S * 3 * ND));
    A(dalloc(&p->h_mask, M));
    A(dalloc(&p->h_drift, NA));
    A(dalloc(&p->h_sexp, nsexp));
    A(dalloc(&p->h_grad, 3 * S * NN));
    A(dalloc(&p->h_cost, S));
    A(dalloc(&p->h_status, 4));
    if (e != cudaSuccess) {
      cudaGetLastError();
      void *ptrs[] = {p->h_maps, p->h_flat, p->h_mask, p->h_drift, p->h_sexp, p->h_grad,
                      p->h_cost, p->h_status};
      for (void *q : ptrs)
        if (q) cudaFree(q);
      p->h_maps = p->h_flat = p->h_mask = p->h_drift = p->h_sexp = p->h_grad = nullptr;
      p->h_cost = nullptr;
      p->h_status = nullptr;
      return EI_ERR_RESOURCE;
    }
  }
  if (!p->h_copy) {   // work + copy streams and events of the host path (created once per plan)
    cudaError_t e = cudaStreamCreateWithFlags(&p->h_copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->h_work, cudaStreamNonBlocking);
    for (int k = 0; k < 4 && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&p->h_ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return EI_ERR_RESOURCE;
    }
  }
  if (p->h_nchunk == 0) setup_chunks(p);
  cudaStream_t st = (cudaStream_t)stream;
  // The whole call (12 copies, a memset, 4-5 kernels) is captured once into a CUDA graph on the
  // plan's work stream and replayed while the arguments stay the same: one launch instead of ~20
  // API calls, which otherwise leave the GPU idle between them (the call is synchronous, so the
  // GPU starts every call idle).  Ordered after the caller's stream by an event; pageable host
  // buffers (not capturable), the timing mode and EI_HOST_GRAPH=0 take the direct path.
  const HostKey key{mu, delta, sigma, flat, mask, drift, s_exp, lambda, cost, g_mu, g_delta, g_sigma, status};
  const char *genv = getenv("EI_HOST_GRAPH");
  // The graph replays DMAs from these exact host addresses, so it is used only while every host
  // buffer is page-locked right now (checked on every call: a freed pinned buffer whose address
  // comes back as pageable memory must not be replayed), and a failed capture disables it only
  // for the arguments that failed
  bool pinned = true;
  for (const void *h : {(const void *)mu, (const void *)delta, (const void *)sigma, (const void *)flat,
                        (const void *)mask, (const void *)drift, (const void *)s_exp, (const void *)cost,
                        (const void *)g_mu, (const void *)g_delta, (const void *)g_sigma, (const void *)status}) {
    if (!h) continue;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess || at.type != cudaMemoryTypeHost) pinned = false;
  }
  cudaGetLastError();
  const bool use_graph = !p->tev && !(genv && atoi(genv) == 0) && pinned &&
                         !(p->h_graph_failed && p->h_fail_key == key);
  if (use_graph) {
    cudaError_t e = cudaEventRecord(p->h_ev[2], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->h_work, p->h_ev[2], 0);
    if (e != cudaSuccess) return EI_ERR_CUDA;
    if (!(p->h_exec && p->h_key == key)) {
      if (p->h_exec) {
        cudaGraphExecDestroy(p->h_exec);
        p->h_exec = nullptr;
      }
      int64_t s0[6];
      for (int i = 0; i < 6; ++i) s0[i] = p->stats[i];
      cudaGraph_t graph = nullptr;
      int rc = EI_ERR_CUDA;
      if (cudaStreamBeginCapture(p->h_work, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        rc = enqueue_host_path(p, mu, delta, sigma, flat, mask, drift, s_exp, lambda, cost, g_mu,
                               g_delta, g_sigma, status, p->h_work);
        if (cudaStreamEndCapture(p->h_work, &graph) != cudaSuccess) rc = EI_ERR_CUDA;
      }
      for (int i = 0; i < 6; ++i) {
        p->h_stats[i] = p->stats[i] - s0[i];
        p->stats[i] = s0[i];
      }
      if (rc == EI_OK && graph && cudaGraphInstantiate(&p->h_exec, graph, 0) == cudaSuccess) {
        p->h_key = key;
      } else {
        p->h_exec = nullptr;
        p->h_graph_failed = true;   // direct path for these arguments
        p->h_fail_key = key;
      }
      if (graph) cudaGraphDestroy(graph);
      cudaGetLastError();
    }
    if (p->h_exec) {
      if (cudaGraphLaunch(p->h_exec, p->h_work) != cudaSuccess) return EI_ERR_CUDA;
      for (int i = 0; i < 6; ++i) p->stats[i] += p->h_stats[i];
      // EI_HOST_SPIN=1 polls an event instead of cudaStreamSynchronize (no measurable difference
      // on the box, where host scheduling noise dominates the 0.2-0.4 ms call)
      const char *spin = getenv("EI_HOST_SPIN");
      if (!(spin && atoi(spin) != 0)) return cudaStreamSynchronize(p->h_work) == cudaSuccess ? EI_OK : EI_ERR_CUDA;
      if (cudaEventRecord(p->h_ev[3], p->h_work) != cudaSuccess) return EI_ERR_CUDA;
      cudaError_t q;
      while ((q = cudaEventQuery(p->h_ev[3])) == cudaErrorNotReady) {
      }
      return q == cudaSuccess ? EI_OK : EI_ERR_CUDA;
    }
  }
  int rc = enqueue_host_path(p, mu, delta, sigma, flat, mask, drift, s_exp, lambda, cost, g_mu,
                             g_delta, g_sigma, status, st);
  if (rc) return rc;
  return cudaStreamSynchronize(st) == cudaSuccess ? EI_OK : EI_ERR_CUDA;
}

}  // extern "C"
