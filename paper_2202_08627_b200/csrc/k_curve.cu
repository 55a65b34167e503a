// k_curve.cu — K2: the fused curve model / residual / cost / dS/dP pass.  SURVEY.md §8(a) a2-a4.
//
// Per detector position (s, theta, t):
//   Delta = z * D P_delta         finite differences along t, halo 1
//   T     = exp(-clamp(P_mu))     eq. 2, clamp R12
//   W^2   = max(w^2 + P_sigma, w^2/100)                 scattering broadening R1, clamp R13
//   s_mod = T A (w/W) exp(-u^2 / 2W^2),  u = m - c - m_o(theta) - Delta   eq. 4 with m_r = 0
//   r     = s_mod - s_exp;  S += r^2                     eq. 5
//   g_mu = -2 sum r s;  g_Delta = 2 sum r s u / W^2;  g_sigma = sum r s (u^2 - W^2) / W^4
//   g_delta = z D^T g_Delta                              halo 1 more (2 in total)
//   dS/dm_o(theta) = sum_t g_Delta(t)                    NEXT-2 (u depends on m_o like on -Delta)
//
// B200 design (DESIGN.md §5 K2): the pass is HBM-bound (s_exp streams once), so it is organised
// for memory-level parallelism rather than per-row CTAs:
//  * work item = one segment of W detector positions of one row (s, theta); a CTA of NT >= W + 4
//    threads evaluates the curve at the W core positions plus a halo of 2 on each side, so D and
//    D^T never need a neighbouring segment (1.5-3 % redundant arithmetic, no extra HBM bytes: the
//    halo loads hit L2/L1);
//  * persistent CTAs own a contiguous run of items (angle fastest, so stepping is a carry chain, no
//    division) and the flat-IC parameters stay in registers; every thread PREFETCHES its loads
//    for the next 2 items (3 projections + 2 neighbours, up to 8 s_exp values) as 4-byte cp.async
//    copies into private shared slots, so each thread keeps ~20 independent loads in flight through
//    its whole life instead of one round trip per row;
//  * one CTA barrier per item: the per-position g values go to a double-buffered shared row, the
//    core threads then write the gradient sinograms directly in K3's PAIR layout (entry
//    e = (g[e-1], g[e]) of every map, pre-multiplied by the Joseph weight dx/|c_dom|);
//  * cost and drift-gradient partials: fp32 per thread (M terms) and per warp (shuffle) -> one
//    partial per (item, warp); K3 sums them in fp64 in index order (fused finalize, K4).
// Deterministic: no float atomics, fixed reduction order, results independent of the grid size.
#include <algorithm>

#include "ei_common.cuh"
#include "tma.cuh"

namespace ei {
namespace {

constexpr int K2_MAXT = 512;   // threads per CTA (max)
constexpr int MPF = 8;         // s_exp values per position held in prefetch registers

// 2^x on the SFU (MUFU.EX2, ~2 ulp): every exponential of the curve model is written as a power
// of two with the log2(e) factor folded into a per-position constant
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr float LOG2E = 1.4426950408889634f;
__device__ __forceinline__ float rcp(float x) {   // MUFU.RCP (~1 ulp), no slow path
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsq(float x) {   // MUFU.RSQ (~2 ulp), no denormal fix-up
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct K2Args {
  const float *P;            // [RS][S][3][NA][ND] (row-split partial projections, summed here)
  int RS, S;
  size_t rstride;            // S * 3 * NA * ND
  const float *flat, *mask, *drift, *s_exp;
  int NA, ND, M, nseg, W;    // W = core positions per segment (<= blockDim - 4)
  int nmap;                  // maps per slice in P: 3 (mu, delta, sigma) or 1 (h, NEXT-3)
  int K;                     // MODES 4, 5: knots of the sampled flat IC (flat = [S][K][ND])
  float zs, inv_du;          // shift factor: z (three-map model) or z gamma (single-map model)
  float *s_mod;              // MODE 0
  float4 *GA;                // MODE 1: pair-layout gradient sinograms (K3 input)
  float2 *GB;
  float2 *GA1;               // MODE 2: pair-layout gradient sinogram of h
  int PADG, RpG;
  const float4 *k3;          // per-angle table, .w = Joseph weight dx/|c_dom|
  float *part_cost, *part_mo;    // [S * NA * nseg * nw] per-warp partials
  int32_t *status;
  int items;                 // S * NA * nseg
};

// prefetch slots per position: P_mu, P_delta(k-1), P_delta(k+1), P_sigma, s_exp[0..MPF); each
// thread's slots are contiguous (stride NQ, odd -> conflict-free), so every slot address is the
// thread's base plus an immediate
constexpr int NQ = 4 + MPF + 1;
constexpr int NSTAGE = 3;      // items in flight per CTA: the current one + 2 prefetched

__device__ __forceinline__ void cp4(uint32_t dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// item position (s, seg, a): angle fastest; a CTA's items are consecutive, so stepping is a carry
// chain (no division), the flat-IC parameters (which depend on (s, t) only) stay in registers and
// the load pointers advance by one row
struct Pos {
  int s, seg, a;
  __device__ __forceinline__ bool step(int NA, int nseg) {   // true: (s, seg) changed
    if (++a < NA) return false;
    a = 0;
    if (++seg == nseg) { seg = 0; ++s; }
    return true;
  }
};

// per-thread load cursor: this thread's position k of item (s, seg, a), as pointers into P and s_exp
struct Cursor {
  const float *pm, *se;   // &P[s][0][a][k], &s_exp[s][a][0][k]
  int k;
  bool valid;
  __device__ __forceinline__ void seek(const K2Args &g, const Pos &q, int t) {
    k = q.seg * g.W - 2 + t;
    valid = k >= 0 && k < g.ND;
    const int plane = g.NA * g.ND;                                 // < 2^30 (plan)
    pm = g.P + (size_t)q.s * g.nmap * plane + (q.a * g.ND + k);
    se = g.s_exp ? g.s_exp + ((size_t)(q.s * g.NA + q.a) * g.M) * g.ND + k : nullptr;
  }
  __device__ __forceinline__ void next_row(const K2Args &g) {     // a -> a + 1, same (s, seg)
    pm += g.ND;
    if (se) se += (size_t)g.M * g.ND;
  }
};

// issue this thread's loads of the cursor's item as 4-byte async copies into its private prefetch
// slots (only this thread reads them: cp.async.wait_group alone orders them — no barrier)
// K2 modes: 0 forward (three maps), 1 cost + gradient (three maps), 2 cost + gradient of the
// paper's single-map model h (NEXT-3: P_mu = P_h, shift z gamma D P_h, no scattering), 3 forward h,
// 4 / 5 cost + gradient / forward of the single-map model with the SAMPLED flat IC (NEXT-4:
// K knots per period per detector pixel, periodic Catmull-Rom, reading R23)
template <int MODE>
struct Mode {
  static constexpr bool cost = MODE == 1 || MODE == 2 || MODE == 4;
  static constexpr bool h = MODE >= 2;
  static constexpr bool sampled = MODE >= 4;
};

template <int MODE>
__device__ __forceinline__ void load_item(const K2Args &g, const Cursor &c, uint32_t slot, int plane,
                                          int dl, int dr) {
  if (!c.valid) return;
  cp4(slot, c.pm);
  if (Mode<MODE>::h) {                 // P_h at k, k-1, k+1
    cp4(slot + 4, c.pm + dl);
    cp4(slot + 8, c.pm + dr);
  } else {                             // P_mu, P_delta(k-1), P_delta(k+1), P_sigma
    cp4(slot + 4, c.pm + plane + dl);
    cp4(slot + 8, c.pm + plane + dr);
    cp4(slot + 12, c.pm + 2 * plane);
  }
  if (Mode<MODE>::cost) {
    const float *se = c.se;
#pragma unroll
    for (int u = 0; u < MPF; ++u) {
      if (u < g.M) cp4(slot + 16 + 4 * u, se);
      se += g.ND;
    }
  }
}

__device__ __forceinline__ float warp_sum(float v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

template <int MODE>
__global__ void __maxnreg__(72) curve_kernel(K2Args g) {
  extern __shared__ __align__(16) float pre_s[];   // [NSTAGE][NQ][NT] prefetch slots
  __shared__ float sgD[2][K2_MAXT], sgm[2][K2_MAXT], sgs[2][K2_MAXT];
  const int NT = blockDim.x;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  const int ND = g.ND;
  int bad = 0, mu_cl = 0, w2_cl = 0;
  float mk[MPF];                                   // mask positions (first MPF) in registers
#pragma unroll
  for (int u = 0; u < MPF; ++u) mk[u] = u < g.M ? __ldg(g.mask + u) : 0.f;
  pdl_wait();   // K1's projections
  // static contiguous split of the items (deterministic, independent of timing)
  const int i0 = (int)(((long long)blockIdx.x * g.items) / gridDim.x);
  const int i1 = (int)(((long long)(blockIdx.x + 1) * g.items) / gridDim.x);
  const int plane = g.NA * ND;
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(pre_s) + 4u * (uint32_t)(t * NQ);
  const uint32_t stage_bytes = 4u * (uint32_t)(NQ * NT);
  Pos cp{i0 / (g.nseg * g.NA), (i0 / g.NA) % g.nseg, i0 % g.NA};   // current item
  Pos lp = cp;                                                       // next item to prefetch
  Cursor lc;
  lc.seek(g, lp, t);
  int dl = lc.k == 0 ? 0 : -1, dr = lc.k == ND - 1 ? 0 : 1;
  auto advance = [&]() {   // lp/lc -> next item
    if (lp.step(g.NA, g.nseg)) {
      lc.seek(g, lp, t);
      dl = lc.k == 0 ? 0 : -1;
      dr = lc.k == ND - 1 ? 0 : 1;
    } else {
      lc.next_row(g);
    }
  };
#pragma unroll
  for (int q = 0; q < NSTAGE - 1; ++q) {
    if (i0 + q < i1) {
      load_item<MODE>(g, lc, slot0 + q * stage_bytes, plane, dl, dr);
      advance();
    }
    cp_commit();
  }
  int fs = -1, fseg = -1;                          // (slice, segment) of the flat registers
  float fA = 0.f, fc = 0.f, fw = 1.f;
  int buf = 0, st = 0;
  for (int item = i0; item < i1; ++item, buf ^= 1, st = (st + 1 == NSTAGE) ? 0 : st + 1,
           cp.step(g.NA, g.nseg)) {
    {   // keep NSTAGE - 1 items in flight: issue item + NSTAGE - 1 into the stage freed last
      const int ns = (st + NSTAGE - 1) % NSTAGE;
      if (item + NSTAGE - 1 < i1) {
        load_item<MODE>(g, lc, slot0 + ns * stage_bytes, plane, dl, dr);
        advance();
      }
      cp_commit();
    }
    const int seg = cp.seg, a = cp.a, s = cp.s;
    const int k = seg * g.W - 2 + t;
    const bool valid = k >= 0 && k < ND;
    const bool core = valid && t >= 2 && t < g.W + 2;
    if (!Mode<MODE>::sampled && valid && (s != fs || seg != fseg)) {   // new (s, seg): A, c, w
      const float *f = g.flat + (size_t)s * 3 * ND + k;
      fA = __ldg(f);
      fc = __ldg(f + ND);
      fw = __ldg(f + 2 * ND);
    }
    fs = s;
    fseg = seg;
    cp_wait<NSTAGE - 1>();   // this item's copies (issued NSTAGE-1 groups ago) have landed
    const float *cur = pre_s + st * NQ * NT + t * NQ;
    const int row = s * g.NA + a;
    float gm = 0.f, gd = 0.f, gs = 0.f, cost = 0.f;
    if (valid) {
      float pm = cur[0], pdl = cur[1], pdr = cur[2], ps = Mode<MODE>::h ? 0.f : cur[3];
      const int kl = k == 0 ? 0 : k - 1, kr = k == ND - 1 ? ND - 1 : k + 1;
      if (g.RS > 1) {   // fixed-order sum of the row-split partials (small problems, L2-resident)
        const int plane = g.NA * ND;
        const float *Pm = g.P + (size_t)s * g.nmap * plane + a * ND;
        const int pd = Mode<MODE>::h ? 0 : plane;   // P_delta plane (the h plane itself)
        for (int r = 1; r < g.RS; ++r) {
          const float *b = Pm + r * g.rstride;
          pm += __ldg(b + k);
          pdl += __ldg(b + pd + kl);
          pdr += __ldg(b + pd + kr);
          if (!Mode<MODE>::h) ps += __ldg(b + 2 * plane + k);
        }
      }
      const float dP = (pdr - pdl) * ((kr - kl == 2 ? 0.5f : 1.f) * g.inv_du);
      const bool mc = (pm > 50.f) || (pm < -50.f);
      pm = fminf(fmaxf(pm, -50.f), 50.f);
      const float T = ex2(-LOG2E * pm);
      float W2 = fmaf(fw, fw, ps);
      const float W2min = 0.01f * fw * fw;
      const bool wc = !Mode<MODE>::sampled && W2 < W2min;
      W2 = wc ? W2min : W2;
      const float invW2 = rcp(W2);
      const float amp = Mode<MODE>::sampled ? T : T * fA * fw * rsq(W2);
      // s = amp exp(-u^2 / 2W^2) = amp 2^(c2 u^2).  (Folding amp into the exponent as log2|amp|
      // saves one FMUL per mask position but adds ~8x the argument rounding and breaks the 1e-3
      // gradient gate at C3's noise level: measured 1.36e-3.)
      const float c2 = -0.5f * LOG2E * invW2;
      const float mo = g.drift ? __ldg(g.drift + a) : 0.f;
      const float base = (Mode<MODE>::sampled ? 0.f : fc) + mo + g.zs * dP;
      if (core) {
        mu_cl += mc;
        w2_cl += wc;
      }
      const size_t rowb = (size_t)row * g.M * ND + k;   // s_exp / s_mod row base
      // per mask position: r = s - s_exp; cost += r^2; with rs = r s:
      //   gmm += rs, gdd += rs u, gq += rs u^2   (g_sigma uses gq - W^2 gmm)
      float gmm = 0.f, gdd = 0.f, gq = 0.f;
      // sampled flat IC of this pixel: knots fsb[q * ND], q = 0..K-1 (periodic Catmull-Rom, R23)
      const float *fsb = Mode<MODE>::sampled ? g.flat + (size_t)s * g.K * ND + k : nullptr;
      auto term = [&](float mpos, int m, float se) {
        const float du_ = mpos - base;
        float sv, tfp = 0.f;   // s, and for the sampled IC T f'(arg)
        float u2 = 0.f;
        if (Mode<MODE>::sampled) {
          const int K = g.K;
          const float x = du_ * (float)K;
          const float fl = floorf(x);
          const float tau = x - fl;
          int i = (int)fl % K;
          if (i < 0) i += K;
          const int q0 = i == 0 ? K - 1 : i - 1, q2 = i + 1 == K ? 0 : i + 1, q3 = q2 + 1 == K ? 0 : q2 + 1;
          const float p0 = __ldg(fsb + q0 * ND), p1 = __ldg(fsb + i * ND), p2 = __ldg(fsb + q2 * ND),
                      p3 = __ldg(fsb + q3 * ND);
          const float a1 = p2 - p0, a2 = fmaf(2.f, p0, fmaf(-5.f, p1, fmaf(4.f, p2, -p3)));
          const float a3 = fmaf(3.f, p1 - p2, p3 - p0);
          const float f = 0.5f * fmaf(tau, fmaf(tau, fmaf(tau, a3, a2), a1), 2.f * p1);
          const float fp = 0.5f * (float)K * fmaf(tau, fmaf(3.f * tau, a3, 2.f * a2), a1);
          sv = amp * f;
          tfp = amp * fp;
        } else {
          u2 = du_ * du_;
          sv = amp * ex2(c2 * u2);
        }
        if (!Mode<MODE>::cost) {
          if (core) g.s_mod[rowb + (size_t)m * ND] = sv;
        } else {
          const float r = sv - se;
          cost = fmaf(r, r, cost);
          const float rsv = r * sv;
          gmm += rsv;
          if (Mode<MODE>::sampled) {
            gdd = fmaf(r, tfp, gdd);   // sum r T f'
          } else {
            gdd = fmaf(rsv, du_, gdd);
            gq = fmaf(rsv, u2, gq);
          }
        }
      };
#pragma unroll
      for (int u = 0; u < MPF; ++u)
        if (u < g.M) term(mk[u], u, Mode<MODE>::cost ? cur[4 + u] : 0.f);   // prefetched s_exp
      for (int m = MPF; m < g.M; ++m)                                                // M > MPF
        term(__ldg(g.mask + m), m, Mode<MODE>::cost ? __ldcs(g.s_exp + rowb + (size_t)m * ND) : 0.f);
      // a non-finite s_exp makes the cost non-finite; only then count the elements (rare path)
      if (Mode<MODE>::cost && core && !isfinite(cost))
        for (int m = 0; m < g.M; ++m) bad += !isfinite(m < MPF ? cur[4 + m] : g.s_exp[rowb + (size_t)m * ND]);
      gm = mc ? 0.f : -2.f * gmm;
      const float gss = fmaf(-W2, gmm, gq);   // sum r s (u^2 - W^2)
      gs = wc ? 0.f : gss * invW2 * invW2;
      gd = Mode<MODE>::sampled ? -2.f * gdd : 2.f * gdd * invW2;   // dS/dShift
    }
    if (Mode<MODE>::cost) {
      sgD[buf][t] = gd;
      sgm[buf][t] = gm;
      sgs[buf][t] = gs;
      // cost and dS/dm_o partials: fp32 per thread (<= M terms) and per warp (32 terms), then
      // fp64 over the warps in warp order
      const float wc_ = warp_sum(core ? cost : 0.f);
      const float wm_ = warp_sum(core ? gd : 0.f);
      if (lane == 0) {   // per-warp partials, (s, a, seg, warp) order; K3 sums them in fp64
        const int pidx = ((s * g.NA + a) * g.nseg + seg) * nw + wid;
        g.part_cost[pidx] = wc_;
        g.part_mo[pidx] = wm_;
      }
      __syncthreads();
      if (t < g.W) {
        const int e = seg * g.W + t;       // pair entry written by this thread
        if (e < ND) {
          const float *D = sgD[buf] + (t + 2 - e);   // D[k] = g_Delta at detector k (window)
          const float zh = 0.5f * g.zs * g.inv_du;
          // g_delta = z D^T g_Delta, D^T written out from the rows of D (a2):
          //   y[j] = [j==0](-g0) + [j==1](g0) + [j==ND-2](-g_{ND-1}) + [j==ND-1](g_{ND-1})
          //        + 1/2 g_{j-1} [1 <= j-1 <= ND-2] - 1/2 g_{j+1} [1 <= j+1 <= ND-2]   (all / du)
          auto gdelta = [&](int j) {
            if (j >= 2 && j <= ND - 3) return zh * (D[j - 1] - D[j + 1]);   // interior rows only
            float y = 0.f;
            if (j == 0) y -= D[0];
            if (j == 1) y += D[0];
            if (j == ND - 2) y -= D[ND - 1];
            if (j == ND - 1) y += D[ND - 1];
            if (j - 1 >= 1 && j - 1 <= ND - 2) y += 0.5f * D[j - 1];
            if (j + 1 >= 1 && j + 1 <= ND - 2) y -= 0.5f * D[j + 1];
            return g.zs * g.inv_du * y;
          };
          const float sc = __ldg(g.k3 + a).w;
          const size_t rb = (size_t)row * g.RpG + g.PADG;
          const float m1 = sgm[buf][t + 2], s1 = sgs[buf][t + 2], d1 = gdelta(e);
          const float m0 = e >= 1 ? sgm[buf][t + 1] : 0.f, s0 = e >= 1 ? sgs[buf][t + 1] : 0.f;
          const float d0 = e >= 1 ? gdelta(e - 1) : 0.f;
          if (Mode<MODE>::h) {   // dS/dP_h = g_mu + z gamma D^T g_Delta (eq. 4 chain rule)
            g.GA1[rb + e] = make_float2(sc * (m0 + d0), sc * (m1 + d1));
            if (e == ND - 1) g.GA1[rb + ND] = make_float2(sc * (m1 + d1), 0.f);
          } else {
            g.GA[rb + e] = make_float4(sc * m0, sc * m1, sc * d0, sc * d1);
            g.GB[rb + e] = make_float2(sc * s0, sc * s1);
            if (e == ND - 1) {   // closing entry e = ND: (g[ND-1], 0)
              g.GA[rb + ND] = make_float4(sc * m1, 0.f, sc * d1, 0.f);
              g.GB[rb + ND] = make_float2(sc * s1, 0.f);
            }
          }
        }
      }
    }
  }
  cp_wait<0>();
  pdl_trigger();
  if (Mode<MODE>::cost) {
    bad = __reduce_add_sync(0xffffffffu, bad);
    mu_cl = __reduce_add_sync(0xffffffffu, mu_cl);
    w2_cl = __reduce_add_sync(0xffffffffu, w2_cl);
    if (lane == 0) {
      if (bad) atomicAdd(&g.status[0], bad);
      if (mu_cl) atomicAdd(&g.status[1], mu_cl);
      if (w2_cl) atomicAdd(&g.status[2], w2_cl);
    }
  }
}

static size_t k2_smem(int NT) { return sizeof(float) * (size_t)NSTAGE * NQ * NT; }

template <int MODE>
cudaError_t launch(const ei_plan &p, const float *flat, const float *mask, const float *drift,
                   const float *s_exp, float *s_mod, int32_t *status, float gamma, cudaStream_t st,
                   int n_knots = 0) {
  K2Args g;
  g.K = n_knots;
  g.P = p.P;
  g.RS = p.proj.RS;
  g.S = p.S;
  g.nmap = Mode<MODE>::h ? 1 : 3;
  g.rstride = (size_t)p.S * g.nmap * p.NA * p.ND;
  g.flat = flat;
  g.mask = mask;
  g.drift = drift;
  g.s_exp = s_exp;
  g.NA = p.NA;
  g.ND = p.ND;
  g.M = p.M;
  g.nseg = p.k2.nseg;
  g.W = p.k2.W;
  g.zs = (float)(p.g.z * (Mode<MODE>::h ? (double)gamma : 1.0));
  g.inv_du = (float)(1.0 / p.g.det_pitch);
  g.s_mod = s_mod;
  g.GA = p.GA;
  g.GB = p.GB;
  g.GA1 = p.GA1;
  g.PADG = p.PADG;
  g.RpG = p.RpG;
  g.k3 = p.tab.k3;
  g.part_cost = p.part_curve;
  g.part_mo = p.part_mo;
  g.status = status;
  g.items = p.S * p.NA * p.k2.nseg;
  const int grid = std::min(g.items, p.k2.ctas);
  const size_t smem = k2_smem(p.k2.NT);
  cudaError_t e = cudaFuncSetAttribute((const void *)curve_kernel<MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(curve_kernel<MODE>, dim3(grid), dim3(p.k2.NT), smem, st, g);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

// K2 launch plan: segments of W = ceil(ND / nseg) positions, nseg the smallest count with
// W + 4 <= 384 threads (balanced segments, <= ~10 % idle threads), CTA = W + 4 rounded up to a
// warp; persistent grid = resident CTAs per SM x SMs.
int plan_curve(ei_plan &p) {
  int nseg = 1;
  while ((p.ND + nseg - 1) / nseg + 4 > 384) ++nseg;
  p.k2.nseg = nseg;
  p.k2.W = (p.ND + nseg - 1) / nseg;
  p.k2.NT = ((p.k2.W + 4 + 31) / 32) * 32;
  p.k2.nw = p.k2.NT / 32;
  if ((long long)p.S * p.NA * nseg > 0x7fffffffLL) return EI_ERR_RESOURCE;   // 32-bit item index
  int dev = 0, sms = 148, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute((const void *)curve_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)k2_smem(p.k2.NT));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, curve_kernel<1>, p.k2.NT, k2_smem(p.k2.NT)) != cudaSuccess || per < 1)
    per = 1;
  cudaGetLastError();
  p.k2.ctas = sms * per;
  return EI_OK;
}

cudaError_t launch_curve_forward(const ei_plan &p, const float *flat, const float *mask,
                                 const float *drift, float *s_mod, cudaStream_t st) {
  return launch<0>(p, flat, mask, drift, nullptr, s_mod, nullptr, 0.f, st);
}

cudaError_t launch_curve_cost_grad(const ei_plan &p, const float *flat, const float *mask,
                                   const float *drift, const float *s_exp, int32_t *status,
                                   cudaStream_t st) {
  return launch<1>(p, flat, mask, drift, s_exp, nullptr, status, 0.f, st);
}

cudaError_t launch_curve_forward_h(const ei_plan &p, float gamma, const float *flat, const float *mask,
                                   const float *drift, float *s_mod, cudaStream_t st) {
  return launch<3>(p, flat, mask, drift, nullptr, s_mod, nullptr, gamma, st);
}

cudaError_t launch_curve_forward_hs(const ei_plan &p, float gamma, const float *fs, int n_knots,
                                    const float *mask, const float *drift, float *s_mod, cudaStream_t st) {
  return launch<5>(p, fs, mask, drift, nullptr, s_mod, nullptr, gamma, st, n_knots);
}

cudaError_t launch_curve_cost_grad_hs(const ei_plan &p, float gamma, const float *fs, int n_knots,
                                      const float *mask, const float *drift, const float *s_exp,
                                      int32_t *status, cudaStream_t st) {
  return launch<4>(p, fs, mask, drift, s_exp, nullptr, status, gamma, st, n_knots);
}

cudaError_t launch_curve_cost_grad_h(const ei_plan &p, float gamma, const float *flat,
                                     const float *mask, const float *drift, const float *s_exp,
                                     int32_t *status, cudaStream_t st) {
  return launch<2>(p, flat, mask, drift, s_exp, nullptr, status, gamma, st);
}

}  // namespace ei
