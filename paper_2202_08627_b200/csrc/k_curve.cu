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
// plus the single-map model of eq. 4 (NEXT-3: P_mu = P_h, Delta = z gamma D P_h, W = w) and its
// sampled-flat variant (NEXT-4: f read by a periodic Catmull-Rom cubic, R23).
//
// B200 design (DESIGN.md §5 K2): the pass is HBM-bound (s_exp streams once), so the loads are
// taken off the compute threads and made deep:
//  * work item = one segment of W detector positions of one row (s, theta); its input is a set of
//    contiguous row pieces — the projections and the M measured curves of that row, W + 8
//    positions each (a halo of 4 on both sides, so D and D^T never need a neighbouring segment);
//  * a producer warp streams each item's row pieces with 1-D bulk copies (TMA engine) into a
//    3-stage shared-memory ring completing on full/empty mbarriers (one elected thread, a handful
//    of copies per item); rows not float4-aligned (N_d % 4 != 0 or misaligned caller arrays) are
//    copied by the producer warp's lanes instead;
//  * consumer thread t owns J = 4 consecutive positions, i.e. one float4 of every staged row
//    (conflict-free LDS.128); the 4 positions are independent chains through the mask loop;
//  * persistent CTAs own a contiguous run of items (angle fastest: the flat parameters of a
//    segment stay in registers across its angles);
//  * per item one consumer barrier: the g values go to a double-buffered shared row, each thread
//    reads its neighbours' float4s for D^T and writes its 4 gradient entries directly in K3's PAIR
//    layout (entry e = (g[e-1], g[e]) of every map, pre-multiplied by the Joseph weight);
//  * cost partials: fp32 per thread, fp64 per warp (shuffle) -> one partial per (item, warp);
//    drift-gradient partials fp32 per warp; K3 sums both in fp64 in index order (fused K4).
// Deterministic: no float atomics, fixed reduction order, results independent of the grid size.
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "ei_common.cuh"
#include "tma.cuh"

namespace ei {
namespace {

#ifdef EI_TRACE
// debug builds only (tools/dbg/step_trace.py): earliest CTA start / latest CTA end of this file's
// kernels in the last traced call (globaltimer, ns)
__device__ unsigned long long g_span_curve[2 * 4];
__device__ __forceinline__ unsigned long long gt_curve() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SPAN_START_curve() const unsigned long long span_t0_ = gt_curve()
#define SPAN_END_curve(k)                                   \
  do {                                                    \
    atomicMin(&g_span_curve[2 * (k)], span_t0_);            \
    atomicMax(&g_span_curve[2 * (k) + 1], gt_curve());         \
  } while (0)
#else
#define SPAN_START_curve()
#define SPAN_END_curve(k)
#endif

constexpr int J = 4;           // detector positions per consumer thread
constexpr int K2_MAXT = 256;   // consumer threads per CTA (max)
constexpr int NST = 3;         // ring stages
constexpr int MPF = 8;         // mask positions kept in registers

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
  const float *P;            // [RS][S][nmap][NA][ND] (row-split partial projections, summed here)
  int RS, S;
  size_t rstride;            // S * nmap * NA * ND
  const float *flat, *mask, *drift, *s_exp;
  int NA, ND, M, nseg, W;    // W = core positions per segment, multiple of 4
  int nmap;                  // maps per slice in P: 3 (mu, delta, sigma) or 1 (h, NEXT-3)
  int nrows;                 // staged rows per item: nmap + M (cost modes) or nmap (forward)
  int WB;                    // staged positions per row: W + 8
  int K;                     // MODES 4, 5: knots of the sampled flat IC (flat = [S][K][ND])
  int vec;                   // 1: rows are 16-B aligned (ND % 4 == 0, aligned arrays) -> TMA
  int vec_smod;              // forward modes: s_mod rows 16-B aligned (float4 stores)
  float zs, inv_du;          // shift factor: z (three-map model) or z gamma (single-map model)
  float *s_mod;              // forward modes
  float4 *GA, *GB;           // MODE 1: triple-layout gradient sinograms (K3 input)
  float *GC;
  float2 *GA1;               // MODES 2, 4: pair-layout gradient sinogram of h
  int PADG, RpG;
  const float4 *k3;          // per-angle table, .w = Joseph weight dx/|c_dom|
  double *part_cost;         // [S * NA * nseg * nw] per-warp cost partials (fp64)
  float *part_mo;            // [S * NA * nseg * nw] per-warp drift-gradient partials
  int32_t *status;
  int items;                 // S * NA * nseg
};

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

// item position (s, seg, a): angle fastest; a CTA's items are consecutive, so stepping is a carry
// chain (no division)
struct Pos {
  int s, seg, a;
  __device__ __forceinline__ void step(int NA, int nseg) {
    if (++a < NA) return;
    a = 0;
    if (++seg == nseg) { seg = 0; ++s; }
  }
};

__device__ __forceinline__ float warp_sum(float v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ float at(const float4 &v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}

// global address of staged row r of item q (rows: maps 0..nmap-1 of P, then the M s_exp rows)
__device__ __forceinline__ const float *row_ptr(const K2Args &g, const Pos &q, int r) {
  const int plane = g.NA * g.ND;                                   // < 2^30 (plan)
  if (r < g.nmap) return g.P + ((size_t)q.s * g.nmap + r) * plane + (size_t)q.a * g.ND;
  return g.s_exp + ((size_t)(q.s * g.NA + q.a) * g.M + (r - g.nmap)) * g.ND;
}

#ifndef EI_K2_MINB
#define EI_K2_MINB 2   // CTAs per SM the register allocation targets (compile-time A/B switch)
#endif
template <int MODE>
__global__ void __launch_bounds__(K2_MAXT + 32, EI_K2_MINB) curve_kernel(K2Args g) {
  extern __shared__ __align__(16) float smem[];   // ring [NST][nrows][WB] + exchange [2][3][WB]
  __shared__ __align__(8) uint64_t full[NST], empty[NST];
  SPAN_START_curve();
  const int NT = blockDim.x - 32;                  // consumer threads
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = NT >> 5;
  const int ND = g.ND, WB = g.WB;
  const int stage_floats = g.nrows * WB;
  float *ring = smem;
  float *xch = smem + NST * stage_floats;         // [2][3][WB]: g_Delta, g_mu, g_sigma rows
  if (t == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], nw);
    }
    mbar_fence_init();
  }
  __syncthreads();
  // static contiguous split of the items (deterministic, independent of timing)
  const int i0 = (int)(((long long)blockIdx.x * g.items) / gridDim.x);
  const int i1 = (int)(((long long)(blockIdx.x + 1) * g.items) / gridDim.x);
  const Pos p0{i0 / (g.nseg * g.NA), (i0 / g.NA) % g.nseg, i0 % g.NA};

  // PDL: only the producer reads K1's output (the projections, via TMA); the consumers' G and
  // partial writes are read only by this call's K3
  if (wid == nw) {   // ---------------- producer warp ----------------
    // the measured curves are inputs, not K1's output: the first item's s_exp rows are requested
    // before the PDL wait, so their HBM latency overlaps K1's tail
    const bool pre0 = g.vec && i0 < i1;
    if (pre0 && lane == 0) {
      const int kb = p0.seg * g.W - J;
      const int ks = max(0, kb), ke = min(ND, kb + WB);
      const uint32_t bytes = (uint32_t)(ke - ks) * 4u;
      mbar_arrive_expect_tx(&full[0], bytes * (uint32_t)g.nrows);   // all rows of the stage
      for (int r = g.nmap; r < g.nrows; ++r)
        bulk_g2s(ring + (ks - kb) + r * WB, row_ptr(g, p0, r) + ks, bytes, &full[0]);
    }
    pdl_wait();   // K1's projections
    Pos q = p0;
    int st = 0;
    uint32_t ph = 0;
    for (int item = i0; item < i1; ++item, q.step(g.NA, g.nseg)) {
      if (item - i0 >= NST) {
        if (lane == 0) mbar_wait(&empty[st], ph ^ 1);
        __syncwarp();
      }
      const int kb = q.seg * g.W - J;                       // position of staged index 0
      const int ks = max(0, kb), ke = min(ND, kb + WB);     // copied positions [ks, ke)
      float *dst = ring + st * stage_floats + (ks - kb);
      if (g.vec) {
        if (lane == 0) {
          const uint32_t bytes = (uint32_t)(ke - ks) * 4u;
          const bool pre = pre0 && item == i0;               // s_exp rows already requested
          if (!pre) mbar_arrive_expect_tx(&full[st], bytes * (uint32_t)g.nrows);
          const int rend = pre ? g.nmap : g.nrows;
          for (int r = 0; r < rend; ++r) bulk_g2s(dst + r * WB, row_ptr(g, q, r) + ks, bytes, &full[st]);
        }
      } else {   // unaligned rows: the warp's lanes copy them
        for (int r = 0; r < g.nrows; ++r) {
          const float *src = row_ptr(g, q, r) + ks;
          for (int k = lane; k < ke - ks; k += 32) dst[r * WB + k] = __ldg(src + k);
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) mbar_arrive(&full[st]);
      }
      if (++st == NST) { st = 0; ph ^= 1; }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  int bad = 0, mu_cl = 0, w2_cl = 0;
  float mk[MPF];                                   // mask positions (first MPF) in registers
#pragma unroll
  for (int u = 0; u < MPF; ++u) mk[u] = u < g.M ? __ldg(g.mask + u) : 0.f;
  int fs = -1, fseg = -1;                          // (slice, segment) of the flat registers
  float4 fA = make_float4(0.f, 0.f, 0.f, 0.f), fc = fA, fw = make_float4(1.f, 1.f, 1.f, 1.f);
  Pos cp = p0;
  int st = 0, buf = 0;
  uint32_t ph = 0;
  for (int item = i0; item < i1; ++item, cp.step(g.NA, g.nseg), buf ^= 1) {
    const int seg = cp.seg, a = cp.a, s = cp.s;
    const int kb = seg * g.W - J;
    const int k0 = kb + J * t;                     // this thread's first position
    const bool staged = J * t < WB;                // inside the staged window (threads are
                                                   // rounded up to a warp)
    const bool any = staged && k0 + J > 0 && k0 < ND;
    if (!Mode<MODE>::sampled && any && (s != fs || seg != fseg)) {   // new (s, seg): flat A, c, w
      const float *f = g.flat + (size_t)s * 3 * ND + k0;
      if (g.vec) {
        fA = __ldg(reinterpret_cast<const float4 *>(f));
        fc = __ldg(reinterpret_cast<const float4 *>(f + ND));
        fw = __ldg(reinterpret_cast<const float4 *>(f + 2 * ND));
      } else {
        float a4[3][J];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int j = 0; j < J; ++j)
            a4[q][j] = (k0 + j >= 0 && k0 + j < ND) ? __ldg(f + q * ND + j) : (q == 2 ? 1.f : 0.f);
        fA = make_float4(a4[0][0], a4[0][1], a4[0][2], a4[0][3]);
        fc = make_float4(a4[1][0], a4[1][1], a4[1][2], a4[1][3]);
        fw = make_float4(a4[2][0], a4[2][1], a4[2][2], a4[2][3]);
      }
    }
    fs = s;
    fseg = seg;
    const int row = s * g.NA + a;
    const float mo = g.drift ? __ldg(g.drift + a) : 0.f;
    if (item == i0) pdl_wait();   // sleep while K1 runs (this CTA may have launched early)
    mbar_wait_full(&full[st], ph);
    const float *stg = ring + st * stage_floats;   // staged rows of this item
    float4 gm4 = make_float4(0.f, 0.f, 0.f, 0.f), gd4 = gm4, gs4 = gm4;
    float cost = 0.f, gmo = 0.f;
    const float4 *r4 = reinterpret_cast<const float4 *>(stg);
    const int W4 = WB / J;
    // D's neighbours outside this thread's float4 of P_delta: from the adjacent lanes (shuffle,
    // all lanes), the warp's edge lanes read the staged row (one lane: no bank conflict)
    const float *pdr = stg + (Mode<MODE>::h ? 0 : WB) + J * t;     // P_delta row at k0
    const float4 Pd0 = staged ? r4[(Mode<MODE>::h ? 0 : W4) + t] : make_float4(0.f, 0.f, 0.f, 0.f);
    float nbl = __shfl_up_sync(0xffffffffu, Pd0.w, 1), nbr = __shfl_down_sync(0xffffffffu, Pd0.x, 1);
    if (lane == 0) nbl = (staged && k0 > 0) ? pdr[-1] : 0.f;
    if (lane == 31) nbr = (staged && k0 + J < ND) ? pdr[J] : 0.f;
    if (any) {
      float4 Pm = Mode<MODE>::h ? Pd0 : r4[t];
      float4 Pd = Pd0;
      float4 Ps = Mode<MODE>::h ? make_float4(0.f, 0.f, 0.f, 0.f) : r4[2 * W4 + t];
      if (g.RS > 1) {   // fixed-order sum of the row-split partials (small problems, L2-resident)
        const int plane = g.NA * ND;
        const float *Pb = g.P + (size_t)s * g.nmap * plane + a * ND + k0;
        const int pdo = Mode<MODE>::h ? 0 : plane;
        // K1B band mode gives RS ~ 10-30 partials: whole float4s where the 4 positions are in the
        // row (k0 is a multiple of 4; rows 16-B aligned), unrolled so the L2 loads overlap; same
        // fixed order r = 1, 2, ... as the scalar path
        int r = 1;
        if (g.vec && k0 >= 0 && k0 + J <= ND) {
          const bool hl = k0 > 0, hr = k0 + J < ND;
#pragma unroll 4
          for (; r < g.RS; ++r) {
            const float *b = Pb + r * g.rstride;
            const float4 v0 = __ldg(reinterpret_cast<const float4 *>(b));
            Pm.x += v0.x; Pm.y += v0.y; Pm.z += v0.z; Pm.w += v0.w;
            if (Mode<MODE>::h) {
              Pd = Pm;
            } else {
              const float4 v1 = __ldg(reinterpret_cast<const float4 *>(b + pdo));
              const float4 v2 = __ldg(reinterpret_cast<const float4 *>(b + 2 * plane));
              Pd.x += v1.x; Pd.y += v1.y; Pd.z += v1.z; Pd.w += v1.w;
              Ps.x += v2.x; Ps.y += v2.y; Ps.z += v2.z; Ps.w += v2.w;
            }
            if (hl) nbl += __ldg(b + pdo - 1);
            if (hr) nbr += __ldg(b + pdo + J);
          }
        }
        for (; r < g.RS; ++r) {
          const float *b = Pb + r * g.rstride;
          float v[3][J];
#pragma unroll
          for (int j = 0; j < J; ++j) {
            const bool ok = k0 + j >= 0 && k0 + j < ND;
            v[0][j] = ok ? __ldg(b + j) : 0.f;
            v[1][j] = ok && !Mode<MODE>::h ? __ldg(b + pdo + j) : 0.f;
            v[2][j] = ok && !Mode<MODE>::h ? __ldg(b + 2 * plane + j) : 0.f;
          }
          Pm.x += v[0][0]; Pm.y += v[0][1]; Pm.z += v[0][2]; Pm.w += v[0][3];
          if (Mode<MODE>::h) {
            Pd = Pm;
          } else {
            Pd.x += v[1][0]; Pd.y += v[1][1]; Pd.z += v[1][2]; Pd.w += v[1][3];
            Ps.x += v[2][0]; Ps.y += v[2][1]; Ps.z += v[2][2]; Ps.w += v[2][3];
          }
          if (k0 > 0) nbl += __ldg(b + pdo - 1);
          if (k0 + J < ND) nbr += __ldg(b + pdo + J);
        }
      }
      const float pdv[J + 2] = {nbl, Pd.x, Pd.y, Pd.z, Pd.w, nbr};   // P_delta at k0-1 .. k0+4
      const float *fsb = Mode<MODE>::sampled ? g.flat + (size_t)s * g.K * ND + k0 : nullptr;
      // per-position constants of the curve (the 4 positions are independent chains: ILP 4)
      float base[J], amp[J], c2[J], W2[J], invW2[J];
      bool mc[J], wc[J], core[J];
      const int segW = seg * g.W, cw = min(g.W, ND - segW);   // core positions [segW, segW + cw)
      const float hf = 0.5f * g.inv_du;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int k = k0 + j;
        const bool ok = (unsigned)k < (unsigned)ND;
        core[j] = (unsigned)(k - segW) < (unsigned)cw;
        // D P_delta (a2): central inside, one-sided at the two ends (selects, no branches)
        const bool lo = k == 0, hi = k == ND - 1;
        const float dP = ((hi ? pdv[j + 1] : pdv[j + 2]) - (lo ? pdv[j + 1] : pdv[j])) * ((lo || hi) ? g.inv_du : hf);
        float pm = at(Pm, j);
        mc[j] = (pm > 50.f) || (pm < -50.f);
        pm = fminf(fmaxf(pm, -50.f), 50.f);
        const float T = ex2(-LOG2E * pm);
        const float w = at(fw, j);
        float w2 = fmaf(w, w, at(Ps, j));
        const float W2min = 0.01f * w * w;
        wc[j] = !Mode<MODE>::sampled && w2 < W2min;
        W2[j] = wc[j] ? W2min : w2;
        invW2[j] = rcp(W2[j]);
        amp[j] = ok ? (Mode<MODE>::sampled ? T : T * at(fA, j) * w * rsq(W2[j])) : 0.f;
        c2[j] = -0.5f * LOG2E * invW2[j];   // exp(-u^2 / 2W^2) = 2^(c2 u^2)
        base[j] = (Mode<MODE>::sampled ? 0.f : at(fc, j)) + mo + g.zs * dP;
        mu_cl += core[j] & mc[j];
        w2_cl += core[j] & wc[j];
      }
      const size_t rowb = (size_t)row * g.M * ND + k0;   // s_mod row base (k0)
      float gmm[J], gdd[J], gq[J], cst[J], smv[J];
#pragma unroll
      for (int j = 0; j < J; ++j) gmm[j] = gdd[j] = gq[j] = cst[j] = 0.f;
      if constexpr (Mode<MODE>::cost && !Mode<MODE>::sampled) {
        // Gaussian flat, cost path: positions (0, 1) and (2, 3) as packed pairs, so every step of
        // the term but the two exponentials is one FADD2 / FMUL2 / FFMA2 (same roundings as the
        // scalar form below):  u = m - base, s = amp 2^(c2 u^2), r = s - s_exp, cost += r^2,
        //   gmm += r s, gdd += r s u, gq += r s u^2
        const float2 nb[2] = {make_float2(-base[0], -base[1]), make_float2(-base[2], -base[3])};
        const float2 am2[2] = {make_float2(amp[0], amp[1]), make_float2(amp[2], amp[3])};
        const float2 cc2[2] = {make_float2(c2[0], c2[1]), make_float2(c2[2], c2[3])};
        const float2 m1 = make_float2(-1.f, -1.f);
        float2 vc[2], vm[2], vd[2], vq[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) vc[h] = vm[h] = vd[h] = vq[h] = make_float2(0.f, 0.f);
        auto term2 = [&](float mpos, const float4 &se4) {
          const float2 mp = make_float2(mpos, mpos);
          const float2 se[2] = {make_float2(se4.x, se4.y), make_float2(se4.z, se4.w)};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float2 du = __fadd2_rn(mp, nb[h]);
            const float2 u2 = __fmul2_rn(du, du);
            const float2 ar = __fmul2_rn(cc2[h], u2);
            const float2 sv = __fmul2_rn(am2[h], make_float2(ex2(ar.x), ex2(ar.y)));
            const float2 r = __ffma2_rn(m1, se[h], sv);
            vc[h] = __ffma2_rn(r, r, vc[h]);
            const float2 rsv = __fmul2_rn(r, sv);
            vm[h] = __fadd2_rn(vm[h], rsv);
            vd[h] = __ffma2_rn(rsv, du, vd[h]);
            vq[h] = __ffma2_rn(rsv, u2, vq[h]);
          }
        };
#pragma unroll
        for (int u = 0; u < MPF; ++u) {          // mask positions in registers
          if (u >= g.M) break;
          term2(mk[u], r4[(g.nmap + u) * W4 + t]);
        }
        for (int m = MPF; m < g.M; ++m) term2(__ldg(g.mask + m), r4[(g.nmap + m) * W4 + t]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          cst[2 * h] = vc[h].x; cst[2 * h + 1] = vc[h].y;
          gmm[2 * h] = vm[h].x; gmm[2 * h + 1] = vm[h].y;
          gdd[2 * h] = vd[h].x; gdd[2 * h + 1] = vd[h].y;
          gq[2 * h] = vq[h].x; gq[2 * h + 1] = vq[h].y;
        }
      } else {
        // one mask position for the 4 positions: r = s - s_exp; cost += r^2; with rs = r s:
        //   gmm += rs, gdd += rs u, gq += rs u^2   (g_sigma uses gq - W^2 gmm)
        auto term = [&](int j, float mpos, int m, float se) {
          const float du_ = mpos - base[j];
          float sv, tfp = 0.f, u2 = 0.f;
          if (Mode<MODE>::sampled) {   // periodic Catmull-Rom through the K knots (R23)
            const int K = g.K;
            const float x = du_ * (float)K;
            const float fl = floorf(x);
            const float tau = x - fl;
            int i = (int)fl % K;
            if (i < 0) i += K;
            const int q0 = i == 0 ? K - 1 : i - 1, q2 = i + 1 == K ? 0 : i + 1, q3 = q2 + 1 == K ? 0 : q2 + 1;
            const bool ok = k0 + j >= 0 && k0 + j < ND;
            const float p0 = ok ? __ldg(fsb + q0 * ND + j) : 0.f, p1 = ok ? __ldg(fsb + i * ND + j) : 0.f,
                        p2 = ok ? __ldg(fsb + q2 * ND + j) : 0.f, p3 = ok ? __ldg(fsb + q3 * ND + j) : 0.f;
            const float a1 = p2 - p0, a2 = fmaf(2.f, p0, fmaf(-5.f, p1, fmaf(4.f, p2, -p3)));
            const float a3 = fmaf(3.f, p1 - p2, p3 - p0);
            const float f = 0.5f * fmaf(tau, fmaf(tau, fmaf(tau, a3, a2), a1), 2.f * p1);
            const float fp = 0.5f * (float)K * fmaf(tau, fmaf(3.f * tau, a3, 2.f * a2), a1);
            sv = amp[j] * f;
            tfp = amp[j] * fp;
          } else {
            u2 = du_ * du_;
            sv = amp[j] * ex2(c2[j] * u2);
          }
          if (!Mode<MODE>::cost) {
            smv[j] = sv;   // stored per mask position below
          } else {
            const float r = sv - se;
            cst[j] = fmaf(r, r, cst[j]);
            const float rsv = r * sv;
            gmm[j] += rsv;
            if (Mode<MODE>::sampled) {
              gdd[j] = fmaf(r, tfp, gdd[j]);   // sum r T f'
            } else {
              gdd[j] = fmaf(rsv, du_, gdd[j]);
              gq[j] = fmaf(rsv, u2, gq[j]);
            }
          }
        };
#pragma unroll
        // forward modes: the 4 positions' s_mod of one mask position as one 16-B store when they
        // are all core positions and the row is 16-B aligned (else element stores)
        const bool allcore = core[0] && core[1] && core[2] && core[3];
        auto store = [&](int m) {
          if (Mode<MODE>::cost) return;
          float *dst = g.s_mod + rowb + (size_t)m * ND;
          if (allcore && g.vec_smod) {
            *reinterpret_cast<float4 *>(dst) = make_float4(smv[0], smv[1], smv[2], smv[3]);
          } else {
#pragma unroll
            for (int j = 0; j < J; ++j)
              if (core[j]) dst[j] = smv[j];
          }
        };
#pragma unroll
        for (int u = 0; u < MPF; ++u) {          // mask positions in registers
          if (u >= g.M) break;
          const float4 se4 = Mode<MODE>::cost ? r4[(g.nmap + u) * W4 + t] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < J; ++j) term(j, mk[u], u, at(se4, j));
          store(u);
        }
        for (int m = MPF; m < g.M; ++m) {        // M > MPF
          const float mp = __ldg(g.mask + m);
          const float4 se4 = Mode<MODE>::cost ? r4[(g.nmap + m) * W4 + t] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int j = 0; j < J; ++j) term(j, mp, m, at(se4, j));
          store(m);
        }
      }
      if (Mode<MODE>::cost) {
        // a non-finite s_exp makes the cost non-finite; only then count the elements (rare)
        if (!isfinite((cst[0] + cst[1]) + (cst[2] + cst[3])))
#pragma unroll
          for (int j = 0; j < J; ++j)
            if (core[j] && !isfinite(cst[j]))
              for (int m = 0; m < g.M; ++m) bad += !isfinite(stg[(g.nmap + m) * WB + J * t + j]);
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const bool ok = (unsigned)(k0 + j) < (unsigned)ND;
          const float gss = fmaf(-W2[j], gmm[j], gq[j]);   // sum r s (u^2 - W^2)
          const float gmj = (mc[j] || !ok) ? 0.f : -2.f * gmm[j];
          const float gsj = (wc[j] || !ok) ? 0.f : gss * invW2[j] * invW2[j];
          const float gdj = !ok ? 0.f : Mode<MODE>::sampled ? -2.f * gdd[j] : 2.f * gdd[j] * invW2[j];
          if (j == 0) { gm4.x = gmj; gs4.x = gsj; gd4.x = gdj; }
          if (j == 1) { gm4.y = gmj; gs4.y = gsj; gd4.y = gdj; }
          if (j == 2) { gm4.z = gmj; gs4.z = gsj; gd4.z = gdj; }
          if (j == 3) { gm4.w = gmj; gs4.w = gsj; gd4.w = gdj; }
          cost += core[j] ? cst[j] : 0.f;
          gmo += core[j] ? gdj : 0.f;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);        // this warp is done with the staged rows
    if (++st == NST) { st = 0; ph ^= 1; }
    if (Mode<MODE>::cost) {
      float4 *x4 = reinterpret_cast<float4 *>(xch + buf * 3 * WB);
      // D^T of a2's D (one-sided end rows) is the central formula y[q] = (g'[q-1] - g'[q+1]) / 2du
      // on a ghost-extended g_Delta: g'[0] = 2 g[0], g'[-1] = -2 g[0], g'[ND-1] = 2 g[ND-1],
      // g'[ND] = -2 g[ND-1], g' = g elsewhere (K2).  Only threads with positions in
      // the row publish; the ghosts outside the row are written by the owners of 0 and ND-1.
      float gx[J];
      if (any) {
        const int jl = ND - 1 - k0;                               // position ND-1 in this float4
        const float gend = (jl >= 0 && jl < J) ? at(gd4, jl) : 0.f;
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int k = k0 + j;
          const float v = at(gd4, j);
          gx[j] = (k == 0 || k == ND - 1) ? 2.f * v : (k == ND ? -2.f * gend : v);
        }
        x4[t] = make_float4(gx[0], gx[1], gx[2], gx[3]);
        x4[W4 + t] = gm4;
        if (!Mode<MODE>::h) x4[2 * W4 + t] = gs4;
        float *xd = xch + buf * 3 * WB - kb;                      // g'_Delta by detector position
        if (k0 == 0) xd[-1] = -2.f * gd4.x;
        if (jl == J - 1) xd[ND] = -2.f * gd4.w;
      }
      // cost partials: fp32 over one thread's 4 positions x M mask positions, fp64 from the warp
      // sum on (so the evaluated cost resolves relative changes far below fp32's 6e-8 x the
      // number of terms: an optimizer's line search compares costs); dS/dm_o partials fp32 per
      // warp; both summed in fp64 over items/warps by K3's finalize
      const double wc_ = warp_sum((double)cost);
      const float wm_ = warp_sum(gmo);
      if (lane == 0) {   // per-warp partials, (s, a, seg, warp) order
        const int pidx = ((s * g.NA + a) * g.nseg + seg) * nw + wid;
        g.part_cost[pidx] = wc_;
        g.part_mo[pidx] = wm_;
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NT) : "memory");   // consumers only
      // K3's input entries of this segment's core, lane-contiguous (consecutive lanes write
      // consecutive entries: fully used store sectors), from the exchange rows, pre-multiplied by
      // the Joseph weight; g_delta[q] = zs D^T g_Delta = (z / 2du) (g'[q-1] - g'[q+1]) on the
      // ghost-extended g'.  Single map: PAIR entries e = (g[e-1], g[e]), e in [segW, segW + cw) and
      // the closing entry N_d after the last segment.  Three maps: TRIPLE entries e = positions
      // e-1, e, e+1 of every map (k_backproject.cu), e in [segW, segW + cw), plus e = -1 before the
      // first and e = N_d after the last segment
      {
        const int segW = seg * g.W, cw = min(g.W, ND - segW);
        const float *xd = xch + buf * 3 * WB - kb;   // g'_Delta by detector position
        const float *xm = xd + WB, *xs = xd + 2 * WB;   // g_mu, g_sigma by detector position
        const float zh = 0.5f * g.zs * g.inv_du;
        const float sc = __ldg(g.k3 + a).w;
        const size_t rb = (size_t)row * g.RpG + g.PADG;
        const int eend = segW + cw + (segW + cw == ND ? 1 : 0);
        if (Mode<MODE>::h) {   // dS/dP_h = g_mu + z gamma D^T g_Delta (eq. 4 chain rule)
          for (int e = segW + t; e < eend; e += NT) {
            const bool lo = e >= 1, hi = e < ND;
            const float m0 = lo ? xm[e - 1] : 0.f, m1 = hi ? xm[e] : 0.f;
            const float d0 = lo ? zh * (xd[e - 2] - xd[e]) : 0.f, d1 = hi ? zh * (xd[e - 1] - xd[e + 1]) : 0.f;
            g.GA1[rb + e] = make_float2(sc * (m0 + d0), sc * (m1 + d1));
          }
        } else {
          auto in = [&](int q) { return (unsigned)q < (unsigned)ND; };
          auto M = [&](int q) { return in(q) ? sc * xm[q] : 0.f; };
          auto Sg = [&](int q) { return in(q) ? sc * xs[q] : 0.f; };
          auto Dl = [&](int q) { return in(q) ? sc * zh * (xd[q - 1] - xd[q + 1]) : 0.f; };
          for (int e = segW - (segW == 0 ? 1 : 0) + t; e < eend; e += NT) {
            g.GA[rb + e] = make_float4(M(e - 1), M(e), Sg(e - 1), Sg(e));
            g.GB[rb + e] = make_float4(Dl(e - 1), Dl(e), M(e + 1), Dl(e + 1));
            g.GC[rb + e] = Sg(e + 1);
          }
        }
      }
    }
  }
  pdl_trigger();
#ifdef EI_TRACE
  asm volatile("bar.sync 2, %0;\n" ::"r"(NT) : "memory");   // consumers only
  if (t == 0) SPAN_END_curve(0);
#endif
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

// dynamic shared memory: the ring (NST stages of nrows rows) + the exchange rows (2 x 3 rows)
static size_t k2_smem(int nrows, int WB) { return sizeof(float) * (size_t)(NST * nrows + 6) * WB; }

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
  g.nrows = g.nmap + (Mode<MODE>::cost ? p.M : 0);
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
  g.WB = p.k2.W + 2 * J;
  auto al = [](const void *q) { return ((uintptr_t)q & 15u) == 0; };
  g.vec = (p.ND % 4 == 0) && al(p.P) && al(flat) && (!s_exp || al(s_exp)) ? 1 : 0;
  g.vec_smod = (p.ND % 4 == 0) && s_mod && al(s_mod) ? 1 : 0;
  g.zs = (float)(p.g.z * (Mode<MODE>::h ? (double)gamma : 1.0));
  g.inv_du = (float)(1.0 / p.g.det_pitch);
  g.s_mod = s_mod;
  g.GA = p.GA;
  g.GB = p.GB;
  g.GC = p.GC;
  g.GA1 = p.GA1;
  g.PADG = p.PADG;
  g.RpG = p.RpG;
  g.k3 = p.tab.k3;
  g.part_cost = p.part_curve;
  g.part_mo = p.part_mo;
  g.status = status;
  g.items = p.S * p.NA * p.k2.nseg;
  const int grid = std::min(g.items, p.k2.ctas);
  const size_t smem = k2_smem(g.nrows, g.WB);
  cudaError_t e = cudaFuncSetAttribute((const void *)curve_kernel<MODE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(curve_kernel<MODE>, dim3(grid), dim3(p.k2.NT + 32), smem, st, g);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

// K2 launch plan: segments of W positions (multiple of 4) with W / 4 + 2 <= 256 consumer threads
// and a staging ring small enough for two CTAs per SM (<= 110 KB; the widest rows still fit one
// CTA); consumers = W / 4 + 2 threads rounded up to a warp, plus the producer warp; persistent
// grid = resident CTAs per SM x SMs.
int plan_curve(ei_plan &p) {
  const int nrows = 3 + p.M;
  auto W_of = [&](int ns) { return (((p.ND + ns - 1) / ns) + 3) & ~3; };
  int nseg = 1;
  const char *mw = getenv("EI_K2_MAXW");   // tuning knob: cap on the segment width
  const int maxw = mw ? std::max(16, atoi(mw)) : 1 << 30;
  // ring small enough for >= 3-4 CTAs per SM (more independent items in flight per SM; measured
  // C4 K2 0.596 -> 0.568 ms at W = 384 vs 768, C3 0.061 -> 0.056 ms at W = 256 vs 512), but
  // segments not narrower than 256 positions (the 8-position halo and per-item costs grow)
  const char *sk = getenv("EI_K2_SMEM_KB");   // tuning knob
  const size_t cap = (size_t)(sk ? std::max(16, atoi(sk)) : 60) * 1024;
  while (W_of(nseg) / J + 2 > K2_MAXT || W_of(nseg) > maxw ||
         (k2_smem(nrows, W_of(nseg) + 2 * J) > cap && W_of(nseg) > 256) ||
         (k2_smem(nrows, W_of(nseg) + 2 * J) > 110 * 1024 && W_of(nseg) > 64))
    ++nseg;
  p.k2.nseg = nseg;
  p.k2.W = W_of(nseg);
  p.k2.NT = ((p.k2.W / J + 2 + 31) / 32) * 32;
  p.k2.nw = p.k2.NT / 32;
  if ((long long)p.S * p.NA * nseg > 0x7fffffffLL) return EI_ERR_RESOURCE;   // 32-bit item index
  if (k2_smem(nrows, p.k2.W + 2 * J) > 220 * 1024) return EI_ERR_SHAPE;      // M too large
  int dev = 0, sms = 148, per = 1;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = k2_smem(nrows, p.k2.W + 2 * J);
  cudaFuncSetAttribute((const void *)curve_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, curve_kernel<1>, p.k2.NT + 32, smem) != cudaSuccess ||
      per < 1)
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

cudaError_t launch_curve_cost_grad_h(const ei_plan &p, float gamma, const float *flat,
                                     const float *mask, const float *drift, const float *s_exp,
                                     int32_t *status, cudaStream_t st) {
  return launch<2>(p, flat, mask, drift, s_exp, nullptr, status, gamma, st);
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

}  // namespace ei

#ifdef EI_TRACE
extern "C" int ei_debug_span_curve(unsigned long long *host, int reset) {
  if (reset) {
    unsigned long long init[8];
    for (int k = 0; k < 4; ++k) { init[2 * k] = ~0ULL; init[2 * k + 1] = 0ULL; }
    return cudaMemcpyToSymbol(ei::g_span_curve, init, sizeof(init)) == cudaSuccess ? 0 : 5;
  }
  return cudaMemcpyFromSymbol(host, ei::g_span_curve, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 5;
}
#endif
