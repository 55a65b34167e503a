// k_project.cu — K1: Joseph ray-driven projection (eq. 1; SURVEY.md §8(a) a1,
// readings R5-R8).  Every angle is handled in its dominant-axis frame: row-dominant angles sample
// the rows of the map, column-dominant angles the rows of the transposed map with (cos, sin)
// swapped (H2); x*(k, i) = (k-(Nd-1)/2)*ic - tn*(i-(N-1)/2) + (N-1)/2, taps (floor x*, +1).
//
// B200 design (DESIGN.md §5 K1):
//  * a CTA owns AGB = 16 consecutive same-dominance angles x RTILE = 64 adjacent rays (32 at four
//    CTAs per SM for single-wave grids and dense wide-window views, plan_projector); it walks the
//    rows in CHUNKS of as many rows as fit a ring stage of E entries (the window of a chunk widens
//    with its rows; narrow where the CTA's rays converge, so chunks there hold more rows); a
//    producer warp streams, with 1-D bulk copies (TMA engine), only the window of PAIR entries (K0
//    layout: entry e = (x[e-1], x[e]) of all maps) that the CTA's rays touch in those rows into a
//    2-3 stage mbarrier ring; every chunk's window is computed exactly on the host (plan) so every
//    index stays inside the staged window without per-sample checks;
//  * a warp = 4 adjacent angles x 8 adjacent rays (angle fastest) or 8 rays x 4 angles (ray
//    fastest, sparse views), chosen per angle group from a bank-conflict model; each thread
//    carries NSL = 4 angle slots (2 for grids far below one wave: 8-angle CTAs);
//  * one tap pair of all three maps = one LDS.128 + one LDS.64; weights (1-w, w) as a float2 and
//    three FFMA2 per sample (acc.x: left taps, acc.y: right taps);
//  * small problems split the rows over RS CTAs (partial P summed in fixed order by K2); the
//    CTAs run work units from a plan table (heaviest first, placed per SM for single waves).
#include <math.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "ei_common.cuh"
#include "tma.cuh"

namespace ei {

// dynamic shared memory of K1: the ring (A plane: 16-B entries for three maps, 8-B for one; B
// plane: 8-B entries, three maps only) and the unit's chunk table
size_t k1_smem(int nst, int E, int nchmax, int nmap) {
  return (size_t)nst * E * (nmap == 3 ? 24 : 8) + (size_t)nchmax * sizeof(int4);
}

namespace {

constexpr int AGB = 16;   // angles per CTA (4 x NSL: 8 with two slots, small grids, plan_projector)
constexpr int RT = 64;    // rays per CTA (RTS = 32 for small single-wave grids, plan_projector)
constexpr int RTS = 32;

template <int NMAP>
struct PL;

template <>
struct PL<3> {
  using A = float4;
  static constexpr bool hasB = true;
};
template <>
struct PL<1> {
  using A = float2;
  static constexpr bool hasB = false;
};

struct ProjArgs {
  const void *MA, *MAT;         // PL<NMAP>::A pairs, [S][N][Rp], entry e at e + PAD (normal / transposed)
  const float2 *MB, *MBT;       // sigma pairs (NMAP = 3), same layout
  const float4 *k1;             // ic, tn, scale, rowdom
  const int2 *groups;           // {first sorted position, count}
  const int *order;             // sorted position -> angle index
  const int *partner;           // angle -> its mirror angle theta + pi, or -1
  const int4 *chunks;           // {cmin, W, first row, rows} per chunk (plan), CSR over units:
  const int *coff;              // [RS][groups][tiles] + 1 offsets into chunks
  const int *unit;              // CTA -> work unit tile + ntile (group + ngroups (rs S + s)) (plan order)
  int N, NA, ND, S, RS, E, nchmax, PAD, Rp, ntile, ngroups;   // E: ring-stage entries
  int nst;                      // ring stages (<= NSTMAX)
  int has_pairs;                // the plan paired mirror angles (else partner[] is all -1)
  float *P;                     // [RS][S][NMAP][NA][ND]
  int *diag;                    // window overflows (ei_plan_info out[4]; must stay 0)
};

#ifdef EI_TRACE
// debug builds only (-DEI_TRACE, tools/dbg/k1_trace.py): per CTA {start ns, end ns, SM id, rows
// with work of its busiest warp}, from %globaltimer
__device__ unsigned long long g_k1_trace[4 * 65536];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

#ifdef EI_TRACE
// debug builds only (tools/dbg/step_trace.py): earliest CTA start / latest CTA end of this file's
// kernels in the last traced call (globaltimer, ns)
__device__ unsigned long long g_span_proj[2 * 4];
__device__ __forceinline__ unsigned long long gt_proj() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SPAN_START_proj() const unsigned long long span_t0_ = gt_proj()
#define SPAN_END_proj(k)                                   \
  do {                                                    \
    atomicMin(&g_span_proj[2 * (k)], span_t0_);            \
    atomicMax(&g_span_proj[2 * (k) + 1], gt_proj());         \
  } while (0)
#else
#define SPAN_START_proj()
#define SPAN_END_proj(k)
#endif

constexpr int NSTMAX = 4;       // pipeline stages (shared-memory ring): 2 (plan), up to 4 (knob)

// Warp-specialised pipeline: warp NCW (the producer) streams each row chunk's window of pair
// entries with 1-D bulk copies (TMA engine) into a NST-deep shared-memory ring, completing on a
// per-stage "full" mbarrier (transaction bytes); the NCW consumer warps wait on "full", compute,
// and release the stage on its "empty" mbarrier.  No CTA-wide barrier inside the loop.
// Map rows are zero-padded by PAD >= the widest window on both sides, so every window is one
// in-bounds contiguous copy per row and plane.  A chunk's rows are staged at a stride of
// (W + 3) & ~1 entries (even: 8-byte-entry rows stay 16-B aligned; >= W + 2: their copy starts at
// the even entry below the window), rows x stride <= E.
// Consumer lane -> (angle aq of the group's current angle quad, ray rq of the warp's 8 rays);
// slot m adds 4m to the angle.  Two mappings, chosen per angle group from a bank-conflict model
// of the geometry (plan_projector): angle fastest (aq = lane & 3, rq = lane >> 2: a quarter warp = 4
// angles x 2 adjacent rays, taps on 2-4 consecutive entries when adjacent angles sample nearly
// the same pixels — dense views) or ray fastest (rq = lane & 7, aq = lane >> 3: a quarter warp =
// 8 adjacent rays of one angle — sparse views with large N, where the 4 angles of a quarter would
// spread over tens of entries and conflict).
// RTILE rays per CTA: RTILE / 8 consumer warps (NT threads) + the producer warp; 2 CTAs per SM
// with 64-ray tiles, 4 with 32-ray tiles (same warps per SM, finer units to balance small grids)
template <int NMAP, int RTILE, int NSL>
__global__ void __launch_bounds__(RTILE * 4 + 32, RTILE == 64 ? 2 : 4) project_kernel(ProjArgs args) {
  constexpr int NT = RTILE * 4, NCW = NT / 32;
  using TA = typename PL<NMAP>::A;
  const int N = args.N, ND = args.ND, E = args.E;
  constexpr bool A8 = sizeof(TA) == 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NST = args.nst;
  TA *sA = reinterpret_cast<TA *>(smem_raw);                                   // [NST][E]
  float2 *sB = reinterpret_cast<float2 *>(sA + NST * E);                     // [NST][E]
  int4 *swin = reinterpret_cast<int4 *>(sB + (NMAP == 3 ? NST * E : 0));     // this unit's chunks
  __shared__ __align__(8) uint64_t full[NSTMAX], empty[NSTMAX];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int un = __ldg(args.unit + blockIdx.x);
  const int tile = un % args.ntile, grp = (un / args.ntile) % args.ngroups, z = un / (args.ntile * args.ngroups);
  const int kt = tile * RTILE;
SPAN_START_proj();
#ifdef EI_TRACE
  const unsigned long long t_start = gtimer();
  __shared__ int s_rows;
  if (tid == 0) s_rows = 0;
  int my_rows = 0;
#endif
  const int2 gr = args.groups[grp];
  const int2 gi = make_int2(gr.x, gr.y & 0xffff);   // {first sorted position, count}
  const bool ray_fast = (gr.y >> 16) != 0;          // lane mapping of this group (plan)
  const int s = z % args.S, rs = z / args.S;
  const float ctr = 0.5f * (float)(N - 1), dctr = 0.5f * (float)(ND - 1);
  const bool rowdom = __ldg(args.k1 + args.order[gi.x]).w != 0.f;
  const size_t Rp = (size_t)args.Rp;
  const TA *gA = reinterpret_cast<const TA *>(rowdom ? args.MA : args.MAT) + (size_t)s * N * Rp + args.PAD;
  const float2 *gB = NMAP == 3 ? (rowdom ? args.MB : args.MBT) + (size_t)s * N * Rp + args.PAD : nullptr;
  const int ui = ((int)rs * args.ngroups + grp) * args.ntile + tile;
  const int cbeg = __ldg(args.coff + ui), nch = __ldg(args.coff + ui + 1) - cbeg;
  const int4 *wtab = args.chunks + cbeg;

  for (int c = tid; c < nch; c += NT + 32) swin[c] = __ldg(wtab + c);
  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NCW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // PDL: only the producer reads K0's output (the packed maps, via TMA); the consumers' prologue
  // (tables, row ranges) overlaps K0's tail and their P writes are read only by this call's K2
  if (w == NCW) {   // ---------------- producer warp ----------------
    pdl_wait();   // K0's packed maps
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int c = 0; c < nch; ++c) {
        if (c >= NST) mbar_wait_sleep(&empty[st], ph ^ 1);
        const int4 wn = swin[c];
        const int i0 = wn.z, rc = wn.w, stride = (wn.y + 3) & ~1;
        const int e0 = wn.x + 1;                       // first staged entry
        const int eb = e0 & ~1, bofs = e0 - eb;        // B plane: 16-B aligned start
        const uint32_t bytes8 = (uint32_t)(((wn.y + bofs) * 8 + 15) & ~15);
        const uint32_t bytesA = A8 ? bytes8 : (uint32_t)wn.y * (uint32_t)sizeof(TA);
        const uint32_t bytesB = NMAP == 3 ? bytes8 : 0u;
        mbar_arrive_expect_tx(&full[st], (uint32_t)rc * (bytesA + bytesB));
        for (int r = 0; r < rc; ++r) {
          const size_t row = (size_t)(i0 + r) * Rp;
          bulk_g2s(sA + st * E + r * stride, gA + row + (A8 ? eb : e0), bytesA, &full[st]);
          if (NMAP == 3) bulk_g2s(sB + st * E + r * stride, gB + row + eb, bytesB, &full[st]);
        }
        if (++st == NST) { st = 0; ph ^= 1; }
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int aq = ray_fast ? lane >> 3 : lane & 3;
  const int k = kt + w * 8 + (ray_fast ? lane & 7 : lane >> 2);
  const float kc = (float)k - dctr;
  float alpha[NSL], tn[NSL], scale[NSL];
  int aidx[NSL];
#pragma unroll
  for (int m = 0; m < NSL; ++m) {
    const int al = min(aq + 4 * m, gi.y - 1);
    const int a = args.order[gi.x + al];
    aidx[m] = (aq + 4 * m < gi.y) ? a : -1;
    const float4 t = __ldg(args.k1 + a);
    alpha[m] = fmaf(kc, t.x, ctr);   // x* = alpha - tn * (i - ctr)
    tn[m] = t.y;
    scale[m] = t.z;
  }
  // warp-uniform row range per slot: rows where at least one lane's ray has a tap inside the
  // map (x* in (-1, N), linear in the row); rows outside it contribute exactly 0
  int wlo[NSL], whi[NSL];
#pragma unroll
  for (int m = 0; m < NSL; ++m) {
    int lo = 0x7fffffff, hi = -0x7fffffff;
    if (aidx[m] >= 0 && k < ND) {
      // x* varies by less than 1/4 entry over the map (e.g. exactly 90 deg, where tn ~ 6e-17 and
      // the row bounds below would overflow int): the ray keeps all rows or none (conservatively
      // wide: rows outside the map read the zero padding inside the staged window)
      if (fabsf(tn[m]) * (float)N < 0.25f) {
        if (alpha[m] > -1.25f && alpha[m] < (float)N + 0.25f) { lo = 0; hi = N - 1; }
      } else {
        float y0 = (alpha[m] + 1.f) / tn[m], y1 = (alpha[m] - (float)N) / tn[m];
        if (y0 > y1) { const float t = y0; y0 = y1; y1 = t; }
        lo = max(0, (int)floorf(y0 + ctr) - 1);
        hi = min(N - 1, (int)ceilf(y1 + ctr) + 1);
      }
    }
    wlo[m] = __reduce_min_sync(0xffffffffu, lo);
    whi[m] = __reduce_max_sync(0xffffffffu, hi);
  }

  float2 am[NSL], ad[NSL], as[NSL];
#pragma unroll
  for (int m = 0; m < NSL; ++m) am[m] = ad[m] = as[m] = make_float2(0.f, 0.f);

  pdl_wait();   // sleep (not spin on the ring) while K0 runs: this CTA may have launched early
  int st = 0;
  uint32_t ph = 0;
  for (int c = 0; c < nch; ++c, st = (st + 1 == NST) ? 0 : st + 1, ph ^= (st == 0)) {
    mbar_wait_full(&full[st], ph);
    const int4 wn = swin[c];
    const int i0 = wn.z, rc = wn.w, i1 = i0 + rc - 1, stride = (wn.y + 3) & ~1;
    bool any = false, all = true;
#pragma unroll
    for (int m = 0; m < NSL; ++m) {
      any |= (whi[m] >= i0 && wlo[m] <= i1);
      all &= (wlo[m] <= i0 && whi[m] >= i1);
    }
    if (any) {
      // staged-window check (the counter behind ei_plan_info out[4]): x* is linear in the row
      // and fmaf / floor are monotone, so every row's tap of a slot lies in the staged entries
      // [wn.x, wn.x + wn.y) iff the chunk's first and last rows' taps do
      {
        const float ya = (float)i0 - ctr, yb = (float)i1 - ctr;
        bool bad = false;
#pragma unroll
        for (int m = 0; m < NSL; ++m) {
          const int ja = __float2int_rd(fmaf(-tn[m], ya, alpha[m]));
          const int jb = __float2int_rd(fmaf(-tn[m], yb, alpha[m]));
          bad |= min(ja, jb) < wn.x || max(ja, jb) >= wn.x + wn.y;
        }
        if (bad) atomicAdd(args.diag, 1);
      }
      const int bofs = (wn.x + 1) & 1;
      const TA *arow = sA + st * E - wn.x + (A8 ? bofs : 0);
      const float2 *brow = sB + st * E - wn.x + bofs;
      float yi = (float)i0 - ctr;
      auto body = [&](bool masked, int i) {
#pragma unroll
        for (int m = 0; m < NSL; ++m) {
          const float xs = fmaf(-tn[m], yi, alpha[m]);
          const int j0 = __float2int_rd(xs);
          const float fr = xs - (float)j0;
          float2 wt = make_float2(1.f - fr, fr);
          if (masked && (i < wlo[m] || i > whi[m])) wt = make_float2(0.f, 0.f);
          const TA va = arow[j0];
          if constexpr (NMAP == 3) {
            am[m] = __ffma2_rn(wt, make_float2(va.x, va.y), am[m]);
            ad[m] = __ffma2_rn(wt, make_float2(va.z, va.w), ad[m]);
            as[m] = __ffma2_rn(wt, brow[j0], as[m]);
          } else {
            am[m] = __ffma2_rn(wt, va, am[m]);
          }
        }
      };
      if (all) {
        for (int r = 0; r < rc; ++r, yi += 1.f, arow += stride, brow += stride) body(false, 0);
      } else {
        for (int r = 0; r < rc; ++r, yi += 1.f, arow += stride, brow += stride) body(true, i0 + r);
      }
#ifdef EI_TRACE
      my_rows += rc;
#endif
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  pdl_trigger();
#ifdef EI_TRACE
  if (lane == 0) atomicMax(&s_rows, my_rows);
  asm volatile("bar.sync 1, %0;\n" ::"r"(NT) : "memory");   // consumers only
  if (tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const size_t b = blockIdx.x;
    if (b < 65536) {
      g_k1_trace[4 * b] = t_start;
      g_k1_trace[4 * b + 1] = gtimer();
      g_k1_trace[4 * b + 2] = smid;
      g_k1_trace[4 * b + 3] = (unsigned long long)s_rows | ((unsigned long long)un << 32);
    }
    SPAN_END_proj(0);
  }
#endif
  if (k >= ND) return;
  const size_t plane = (size_t)args.NA * ND;
  float *out = args.P + ((size_t)rs * args.S + s) * NMAP * plane + k;
  float *outm = out + (ND - 1 - 2 * k);   // mirrored detector position ND-1-k
#pragma unroll
  for (int m = 0; m < NSL; ++m) {
    if (aidx[m] < 0) continue;
    const float v0 = (am[m].x + am[m].y) * scale[m];
    out[(size_t)aidx[m] * ND] = v0;
    // the mirror angle theta + pi samples the same line at the mirrored detector position
    // (R6: detector centred), so its projection is this value: one projection, two rows
    const int b = args.has_pairs ? __ldg(args.partner + aidx[m]) : -1;   // no load in the tail
    if (b >= 0) outm[(size_t)b * ND] = v0;
    if constexpr (NMAP == 3) {
      const float v1 = (ad[m].x + ad[m].y) * scale[m], v2 = (as[m].x + as[m].y) * scale[m];
      out[plane + (size_t)aidx[m] * ND] = v1;
      out[2 * plane + (size_t)aidx[m] * ND] = v2;
      if (b >= 0) {
        outm[plane + (size_t)b * ND] = v1;
        outm[2 * plane + (size_t)b * ND] = v2;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Band mode (K1B, small maps: C1, C2, P1; DESIGN.md §5 K1B).  The per-tile units above differ in
// work by up to 128 rows (detector-end tiles and near-axis angles miss much of the map), and on a
// single-wave grid the step ends with its heaviest unit.  Here a unit is (angle group, band of BR
// map rows, slice): the producer stages the band's FULL rows once (entries -2 .. N+1 of the pair
// layout, one bulk copy per row and plane), and the consumer warps sweep ALL rays over it, 64 per
// pass.  Every map row meets about the same number of rays ((N+1)|c_dom| per angle), so the units
// carry nearly equal work, and one staged byte serves every ray of the group that crosses it.  The
// band's sum is a partial projection P[band]; K2 adds the bands in fixed order (as for RS).  A tap
// index outside the map is clamped onto the zero entries -1 / N+1, which contribute exactly 0.
constexpr int NCWB = 8;   // consumer warps per band CTA (64 rays per pass)

struct BandArgs {
  const void *MA, *MAT;         // PL<NMAP>::A pairs, [S][N][Rp], entry e at e + PAD
  const float2 *MB, *MBT;       // sigma pairs (NMAP = 3)
  const float4 *k1;
  const int2 *groups;
  const int *order, *partner;
  int N, NA, ND, S, BR, nbands, ngroups, PAD, Rp, stride, has_pairs;
  float *P;                     // [nbands][S][NMAP][NA][ND]
};

size_t k1_band_smem(int BR, int stride, int nmap) {
  return (size_t)BR * stride * (nmap == 3 ? 24 : 8);
}

template <int NMAP, int NSLB>
__global__ void __launch_bounds__(NCWB * 32 + 32, 2) project_band_kernel(BandArgs args) {
  constexpr int NT = NCWB * 32;
  using TA = typename PL<NMAP>::A;
  const int N = args.N, ND = args.ND, stride = args.stride;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  TA *sA = reinterpret_cast<TA *>(smem_raw);                            // [BR][stride]
  float2 *sB = reinterpret_cast<float2 *>(sA + (size_t)args.BR * stride);  // [BR][stride] (NMAP 3)
  __shared__ __align__(8) uint64_t full;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int grp = blockIdx.x % args.ngroups;
  const int band = (blockIdx.x / args.ngroups) % args.nbands;
  const int s = blockIdx.x / (args.ngroups * args.nbands);
  const int i0 = band * args.BR, rc = min(args.BR, N - i0);
  SPAN_START_proj();
  const int2 gr = args.groups[grp];
  const int2 gi = make_int2(gr.x, gr.y & 0xffff);
  const bool ray_fast = (gr.y >> 16) != 0;
  const float ctr = 0.5f * (float)(N - 1), dctr = 0.5f * (float)(ND - 1);
  const bool rowdom = __ldg(args.k1 + args.order[gi.x]).w != 0.f;
  const size_t Rp = (size_t)args.Rp;
  if (tid == 0) {
    mbar_init(&full, 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (w == NCWB) {   // ---------------- producer warp: the band's rows, entries -2 .. N+1 ----------------
    pdl_wait();   // K0's packed maps
    if (lane == 0) {
      const TA *gA = reinterpret_cast<const TA *>(rowdom ? args.MA : args.MAT) + (size_t)s * N * Rp + args.PAD - 2;
      const float2 *gB = NMAP == 3 ? (rowdom ? args.MB : args.MBT) + (size_t)s * N * Rp + args.PAD - 2 : nullptr;
      const uint32_t bytesA = (uint32_t)(((size_t)(N + 4) * sizeof(TA) + 15) & ~(size_t)15);
      const uint32_t bytesB = NMAP == 3 ? (uint32_t)(((N + 4) * 8 + 15) & ~15) : 0u;
      mbar_arrive_expect_tx(&full, (uint32_t)rc * (bytesA + bytesB));
      for (int r = 0; r < rc; ++r) {
        const size_t row = (size_t)(i0 + r) * Rp;
        bulk_g2s(sA + (size_t)r * stride, gA + row, bytesA, &full);
        if (NMAP == 3) bulk_g2s(sB + (size_t)r * stride, gB + row, bytesB, &full);
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int aq = ray_fast ? lane >> 3 : lane & 3, rq = ray_fast ? lane & 7 : lane >> 2;
  float tn[NSLB];
  int ang[NSLB];   // the slot's angle (clamped to the group's last for idle slots)
  bool live[NSLB];
#pragma unroll
  for (int m = 0; m < NSLB; ++m) {
    const int al = min(aq + 4 * m, gi.y - 1);
    ang[m] = args.order[gi.x + al];
    live[m] = aq + 4 * m < gi.y;
    tn[m] = __ldg(args.k1 + ang[m]).y;
  }
  const float ya = (float)i0 - ctr, yb = ya + (float)(rc - 1);
  const size_t plane = (size_t)args.NA * ND;
  float *outb = args.P + ((size_t)band * args.S + s) * NMAP * plane;
  const TA *arow0 = sA + 2;                 // entry 0 of row 0 (entry e at index e + 2)
  const float2 *brow0 = sB + 2;
  pdl_wait();   // sleep (not spin on the barrier) while K0 runs
  mbar_wait_full(&full, 0);
  for (int kt = 0; kt < ND; kt += NCWB * 8) {
    const int k = kt + w * 8 + rq;
    const float kc = (float)k - dctr;
    float alpha[NSLB];
    bool hit = false;
#pragma unroll
    for (int m = 0; m < NSLB; ++m) {
      alpha[m] = fmaf(kc, __ldg(args.k1 + ang[m]).x, ctr);   // x* = alpha - tn * (i - ctr)
      const float xa = fmaf(-tn[m], ya, alpha[m]), xb = fmaf(-tn[m], yb, alpha[m]);
      hit |= live[m] && k < ND && fmaxf(xa, xb) > -1.f && fminf(xa, xb) < (float)N;
    }
    float2 am[NSLB], ad[NSLB], as[NSLB];
#pragma unroll
    for (int m = 0; m < NSLB; ++m) am[m] = ad[m] = as[m] = make_float2(0.f, 0.f);
    if (__any_sync(0xffffffffu, hit)) {   // some ray of the warp crosses the band inside the map
      const TA *arow = arow0;
      const float2 *brow = brow0;
      float yi = ya;
      for (int r = 0; r < rc; ++r, yi += 1.f, arow += stride, brow += stride) {
#pragma unroll
        for (int m = 0; m < NSLB; ++m) {
          const float xs = fmaf(-tn[m], yi, alpha[m]);
          const int j0 = __float2int_rd(xs);
          const float fr = xs - (float)j0;
          const float2 wt = make_float2(1.f - fr, fr);
          const int e = min(max(j0 + 1, -1), N + 1);   // tap pair (x[j0], x[j0+1]) = entry j0 + 1
          const TA va = arow[e];
          if constexpr (NMAP == 3) {
            am[m] = __ffma2_rn(wt, make_float2(va.x, va.y), am[m]);
            ad[m] = __ffma2_rn(wt, make_float2(va.z, va.w), ad[m]);
            as[m] = __ffma2_rn(wt, brow[e], as[m]);
          } else {
            am[m] = __ffma2_rn(wt, va, am[m]);
          }
        }
      }
    }
    if (k < ND) {
      float *out = outb + k, *outm = outb + (ND - 1 - k);
#pragma unroll
      for (int m = 0; m < NSLB; ++m) {
        if (!live[m]) continue;
        const int a = ang[m];
        const float scale = __ldg(args.k1 + a).z;
        const int b = args.has_pairs ? __ldg(args.partner + a) : -1;
        const float v0 = (am[m].x + am[m].y) * scale;
        out[(size_t)a * ND] = v0;
        if (b >= 0) outm[(size_t)b * ND] = v0;
        if constexpr (NMAP == 3) {
          const float v1 = (ad[m].x + ad[m].y) * scale, v2 = (as[m].x + as[m].y) * scale;
          out[plane + (size_t)a * ND] = v1;
          out[2 * plane + (size_t)a * ND] = v2;
          if (b >= 0) {
            outm[plane + (size_t)b * ND] = v1;
            outm[2 * plane + (size_t)b * ND] = v2;
          }
        }
      }
    }
  }
  pdl_trigger();
#ifdef EI_TRACE
  asm volatile("bar.sync 1, %0;\n" ::"r"(NT) : "memory");   // consumers only
  if (tid == 0) SPAN_END_proj(0);
#endif
}

template <int NMAP>
cudaError_t launch_band(const ei_plan &p, float *P, cudaStream_t st) {
  BandArgs a;
  if (NMAP == 3) {
    a.MA = p.MA; a.MAT = p.MAT; a.MB = p.MB; a.MBT = p.MBT;
  } else {
    a.MA = p.M1; a.MAT = p.M1T; a.MB = nullptr; a.MBT = nullptr;
  }
  a.k1 = p.tab.k1;
  a.groups = p.proj.groups;
  a.order = p.proj.order;
  a.partner = p.proj.partner;
  a.has_pairs = p.npairs > 0 ? 1 : 0;
  a.N = p.N; a.NA = p.NA; a.ND = p.ND; a.S = p.S;
  a.BR = p.proj.BR; a.nbands = p.proj.RS; a.ngroups = p.proj.n_groups;
  a.PAD = p.proj.PAD; a.Rp = p.proj.Rp; a.stride = p.proj.bstride;
  a.P = P;
  const size_t smem = k1_band_smem(a.BR, a.stride, NMAP);
  auto kern = p.proj.nsl == 2 ? project_band_kernel<NMAP, 2> : project_band_kernel<NMAP, 4>;
  cudaError_t e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.proj.n_groups * p.proj.RS * p.S);
  e = launch_pdl(kern, grid, dim3(NCWB * 32 + 32), smem, st, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int NMAP>
cudaError_t launch(const ei_plan &p, int RS, float *P, cudaStream_t st) {
  if (p.proj.band && RS == p.proj.RS) return launch_band<NMAP>(p, P, st);
  ProjArgs a;
  if (NMAP == 3) {
    a.MA = p.MA; a.MAT = p.MAT; a.MB = p.MB; a.MBT = p.MBT;
  } else {
    a.MA = p.M1; a.MAT = p.M1T; a.MB = nullptr; a.MBT = nullptr;
  }
  a.k1 = p.tab.k1;
  a.groups = p.proj.groups;
  a.order = p.proj.order;
  a.partner = p.proj.partner;
  a.has_pairs = p.npairs > 0 ? 1 : 0;
  a.chunks = RS == 1 ? p.proj.chunks1 : p.proj.chunksRS;
  a.coff = RS == 1 ? p.proj.coff1 : p.proj.coffRS;
  a.unit = RS == 1 ? p.proj.unit1 : p.proj.unitRS;
  a.ntile = p.proj.n_tiles;
  a.ngroups = p.proj.n_groups;
  a.N = p.N; a.NA = p.NA; a.ND = p.ND; a.S = p.S; a.RS = RS; a.E = p.proj.E;
  a.PAD = p.proj.PAD; a.Rp = p.proj.Rp;
  a.nchmax = RS == 1 ? p.proj.nchmax1 : p.proj.nchmaxRS;
  a.P = P;
  a.diag = p.diag;
  a.nst = p.proj.nst;
  const size_t smem = k1_smem(a.nst, a.E, a.nchmax, NMAP);
  auto kern = p.proj.nsl == 2 ? (p.proj.RT == RT ? project_kernel<NMAP, RT, 2> : project_kernel<NMAP, RTS, 2>)
                                : (p.proj.RT == RT ? project_kernel<NMAP, RT, 4> : project_kernel<NMAP, RTS, 4>);
  cudaError_t e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (RS != 1 && RS != p.proj.RS) return cudaErrorInvalidValue;   // unit tables exist for these
  dim3 grid(p.proj.n_tiles * p.proj.n_groups * p.S * RS);
  e = launch_pdl(kern, grid, dim3(p.proj.RT * 4 + 32), smem, st, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

// Host planning for K1 (called once by ei_plan_create):
//  * groups: runs of <= AGB angularly adjacent angles of one dominance class;
//  * chunk table: for every (row split, group, ray tile) the rows are cut greedily into chunks of
//    as many rows as fit one ring stage of E entries at a stride of (W + 3) & ~1 per row (<= RCMAX
//    rows), where W is the width of the chunk's window of pair entries: from the fp64 positions of
//    the extreme rays at every row (x* is linear in ray and row), widened by one entry on each side
//    so fp32 rounding in the kernel can never leave the window; rows whose window misses the map
//    contribute nothing and get no chunk.  Stored {first entry - 1, W, first row, rows} in CSR form
//    (offsets per unit);
//  * the ring stage size E from the shared-memory budget, and the row split RS of the cost path for
//    problems with fewer than ~2 CTAs per SM.
struct Chunks {
  std::vector<int4> c;      // all chunks, unit by unit
  std::vector<int> off;     // [RS][groups][tiles] + 1
  int nchmax = 0, wmax = 1, rcmax = 0;
  long long rows(size_t u) const {   // rows staged by unit u (its cost)
    long long r = 0;
    for (int q = off[u]; q < off[u + 1]; ++q) r += c[q].w;
    return r;
  }
};

static bool build_chunks(const ei_plan &p, const double *angles, const std::vector<int2> &groups,
                         const std::vector<int> &order, int RS, int E, int RCMAX, Chunks &ch) {
  const int N = p.N, ND = p.ND;
  const double dx = p.g.pixel, du = p.g.det_pitch, ctr = 0.5 * (N - 1), dctr = 0.5 * (ND - 1);
  const int rt = p.proj.RT, ntile = (ND + rt - 1) / rt;
  ch = Chunks();
  ch.off.push_back(0);
  std::vector<double> lo(N), hi(N);
  for (int rs = 0; rs < RS; ++rs) {
    const int r0 = (int)(((long long)rs * N) / RS), r1 = (int)(((long long)(rs + 1) * N) / RS);
    for (size_t g = 0; g < groups.size(); ++g) {
      for (int t = 0; t < ntile; ++t) {
        const int kt = t * rt;
        // per-row extreme floor(x*) over the group's angles and the tile's extreme rays
        for (int i = r0; i < r1; ++i) {
          lo[i] = 1e300;
          hi[i] = -1e300;
        }
        for (int q = 0; q < groups[g].y; ++q) {
          const int a = order[groups[g].x + q];
          const double cs = cos(angles[a]), sn = sin(angles[a]);
          const bool rd = fabs(cs) >= fabs(sn);
          const double cd = rd ? cs : sn, so = rd ? sn : cs;
          for (int kk : {kt, kt + rt - 1}) {
            const double a0 = (kk - dctr) * du / (cd * dx) + ctr, b0 = so / cd;
            for (int i = r0; i < r1; ++i) {
              const double xs = floor(a0 - b0 * (i - ctr));
              lo[i] = std::min(lo[i], xs);
              hi[i] = std::max(hi[i], xs);
            }
          }
        }
        int i = r0;
        while (i < r1) {
          if (hi[i] + 1 < -1 || lo[i] - 1 > N - 1) { ++i; continue; }   // taps [lo-1, hi+1] miss the map
          double clo = lo[i], chi = hi[i];
          int rc = 1;
          const int W1 = (int)(chi - clo) + 3;
          if ((((W1 + 3) & ~1)) > E) return false;                      // one row must fit a stage
          while (i + rc < r1 && rc < RCMAX) {
            const int j = i + rc;
            if (hi[j] + 1 < -1 || lo[j] - 1 > N - 1) break;
            const double nlo = std::min(clo, lo[j]), nhi = std::max(chi, hi[j]);
            const int W = (int)(nhi - nlo) + 3;
            if ((long long)(rc + 1) * ((W + 3) & ~1) > E) break;
            clo = nlo;
            chi = nhi;
            ++rc;
          }
          const int W = (int)(chi - clo) + 3;
          ch.c.push_back(make_int4((int)clo - 1, W, i, rc));
          ch.wmax = std::max(ch.wmax, W);
          ch.rcmax = std::max(ch.rcmax, rc);
          i += rc;
        }
        const int n = (int)ch.c.size() - ch.off.back();
        ch.nchmax = std::max(ch.nchmax, n);
        ch.off.push_back((int)ch.c.size());
      }
    }
  }
  return true;
}

// Shared-memory wavefront model of the consumer gathers for one lane mapping (see the kernel):
// per quarter warp the LDS.128 of the A plane costs the largest number of distinct 16-B entries
// falling on one bank group (entry mod 8); per half warp the LDS.64 of the B plane the largest
// number of distinct 8-B entries per bank pair (entry mod 16).  Averaged over sampled (ray tile,
// warp, slot, row) positions of angle group g.
static double wavefront_model(const ei_plan &p, const double *angles, const std::vector<int2> &groups,
                              const std::vector<int> &order, size_t g, bool ray_fast) {
  const int N = p.N, ND = p.ND;
  const double dx = p.g.pixel, du = p.g.det_pitch, ctr = 0.5 * (N - 1), dctr = 0.5 * (ND - 1);
  double wf = 0.0;
  long long n = 0;
  const int rows[5] = {0, N / 4, N / 2, (3 * N) / 4, N - 1};
  const int tstep = std::max(1, (ND / 64) / 6);
  for (int kt = 0; kt + 64 <= ND; kt += 64 * tstep)
      for (int w = 0; w < 8; ++w)
        for (int m = 0; m < p.proj.nsl; ++m)
          for (int i : rows) {
            long long e[32];
            for (int lane = 0; lane < 32; ++lane) {
              const int aq = ray_fast ? lane >> 3 : lane & 3, rq = ray_fast ? lane & 7 : lane >> 2;
              const int al = std::min(aq + 4 * m, groups[g].y - 1);
              const double th = angles[order[groups[g].x + al]];
              const double cs = cos(th), sn = sin(th);
              const bool rd = fabs(cs) >= fabs(sn);
              const double cd = rd ? cs : sn, so = rd ? sn : cs;
              const int k = kt + 8 * w + rq;
              const double xs = (k - dctr) * du / (cd * dx) - (so / cd) * (i - ctr) + ctr;
              e[lane] = (long long)floor(xs) + 1;
            }
            auto cost = [&](int lanes, int banks) {
              int tot = 0;
              for (int q0 = 0; q0 < 32; q0 += lanes) {
                int worst = 1;
                for (int b = 0; b < banks; ++b) {
                  long long seen[32];
                  int ns = 0;
                  for (int l = q0; l < q0 + lanes; ++l) {
                    if ((((e[l] % banks) + banks) % banks) != b) continue;
                    bool dup = false;
                    for (int z = 0; z < ns; ++z) dup |= seen[z] == e[l];
                    if (!dup) seen[ns++] = e[l];
                  }
                  worst = std::max(worst, ns);
                }
                tot += worst;
              }
              return tot;
            };
            wf += cost(8, 8) + cost(16, 16);
            ++n;
          }
  return n ? wf / n : 0.0;
}

// Launch order of the K1 work units (tile, group, row split, slice).  Unit cost = rows of its
// staged chunks (W > 0; the ray tiles at the detector ends and near-axis angles have few).
//  * Grid within one wave (units <= 2 CTAs x SMs): the block scheduler places block b and block
//    b + SMs on the same SM (measured, tools/dbg/k1_trace.py: C2 SM 120 ran blocks 138 and 286),
//    and the SM's time is the sum of its two CTAs' work.  So the heaviest units run alone on the
//    SMs that get one CTA, and the rest are paired heaviest with lightest.
//  * Larger grids: heaviest first (longest-processing-time order), so the light units fill the
//    tail of the last wave; slice by slice, so the CTAs in flight share one slice's map in L2
//    (LPT across all 64 slices of C4 raised K1's DRAM traffic from ~18 to ~170 MB per slice).
static std::vector<int> order_units(const Chunks &ch, int RS, int n_groups, int ntile, int S, int cps) {
  const int nu1 = RS * n_groups * ntile;          // per slice: (rs, group, tile)
  std::vector<std::pair<long long, int>> cost;   // (slice, -cost) key, unit
  cost.reserve((size_t)nu1 * S);
  for (int s = 0; s < S; ++s)
    for (int rs = 0; rs < RS; ++rs)
      for (int g = 0; g < n_groups; ++g)
        for (int t = 0; t < ntile; ++t) {
          const long long c = ch.rows(((size_t)rs * n_groups + g) * ntile + t);
          cost.push_back({(long long)s * (1LL << 40) - c, t + ntile * (g + n_groups * (rs * S + s))});
        }
  std::stable_sort(cost.begin(), cost.end());    // slice-major, heaviest first; ties keep (rs, g, t)
  const int n = (int)cost.size();
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  std::vector<int> unit(n);
  if (n > sms && n <= cps * sms && !getenv("EI_K1_LPT")) {
    // one wave: SM m holds blocks m, m + sms, ...; each unit (heaviest first) goes to the SM with
    // the least work so far among those with a free block
    std::vector<int> cap(sms, 0), used(sms, 0);
    std::vector<long long> load(sms, 0);
    for (int b = 0; b < n; ++b) cap[b % sms] += 1;
    for (int q = 0; q < n; ++q) {
      int best = -1;
      for (int m = 0; m < sms; ++m)
        if (used[m] < cap[m] && (best < 0 || load[m] < load[best])) best = m;
      unit[best + used[best] * sms] = cost[q].second;
      used[best] += 1;
      long long rows = (-cost[q].first) % (1LL << 40);   // the unit's rows (key = s 2^40 - rows)
      if (rows < 0) rows += 1LL << 40;
      load[best] += rows;
    }
  } else {
    for (int b = 0; b < n; ++b) unit[b] = cost[b].second;
  }
  return unit;
}

int plan_projector(ei_plan &p, const double *angles, const std::vector<int> &proj_angles,
                   std::vector<int2> &groups, std::vector<int> &order, std::vector<int4> &chunks1,
                   std::vector<int> &coff1, std::vector<int4> &chunksRS, std::vector<int> &coffRS,
                   std::vector<int> &unit1, std::vector<int> &unitRS) {
  const int N = p.N, ND = p.ND;
  const int NA = (int)proj_angles.size();   // the angles K1 projects (mirror pairs: primaries)
  // groups = runs of angularly adjacent angles (sorted by angle mod 2 pi) of one dominance class
  std::vector<int> idx(proj_angles);
  auto wrap = [](double t) { t = fmod(t, 2 * M_PI); return t < 0 ? t + 2 * M_PI : t; };
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return wrap(angles[x]) < wrap(angles[y]); });
  auto rowdom = [&](int a) { return fabs(cos(angles[a])) >= fabs(sin(angles[a])); };
  // Angles per CTA: 16 (4 slots per thread), or 8 (2 slots) when the 16-angle grid of 64-ray
  // tiles would leave more than half the SMs idle: twice the units, each half as long (C1 K1 11.9
  // -> 10.6 us, step 27.9 -> 26.8; P1 unchanged; on C2's single wave of 138 x 4 units the 8-angle
  // units lose more in per-unit staging than they gain in balance, K1 33.1 -> 37.2 us, so C2
  // keeps 16; tools/dbg/sweep_nsl.sh; knob EI_K1_NSL)
  int sms0 = 148, dev0 = 0;
  if (cudaGetDevice(&dev0) == cudaSuccess) cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
  cudaGetLastError();
  p.proj.nsl = 2LL * ((ND + RT - 1) / RT) * ((NA + AGB - 1) / AGB) * p.S <= sms0 ? 2 : 4;
  if (const char *e = getenv("EI_K1_NSL")) p.proj.nsl = atoi(e) == 2 ? 2 : 4;   // tuning knob
  const int agb = 4 * p.proj.nsl;
  order.clear();
  groups.clear();
  for (int q = 0; q < NA; ++q) {
    const int a = idx[q];
    if (groups.empty() || groups.back().y == agb || rowdom(a) != rowdom(order.back()))
      groups.push_back(make_int2((int)order.size(), 0));
    order.push_back(a);
    groups.back().y += 1;
  }
  const size_t per_entry = 24;          // float4 + float2 per staged entry
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  // Staging ring: 2 stages of E entries, within a shared-memory budget that keeps two (64-ray
  // tiles) or four (32-ray tiles) CTAs per SM (104 / 50 KB, knob EI_K1_SMEM_KB), filled by chunks
  // of as many rows as fit a stage (<= RCMAX, which leaves every CTA >= 2 chunks).  First the row
  // split RS from the rows per chunk a 4-stage ring would allow; fewer, larger chunks cost less
  // per-chunk synchronisation than a deeper ring (measured vs the 4-stage ring: C4 K1 9.16 -> 8.67
  // ms, C3 0.71 -> 0.62, C5 1.39 -> 1.23, P1 40.5 -> 39.2 us per evaluation; 3 stages where they
  // fit: P1 40.7), and chunks sized by their own window rather than the widest one hold more rows
  // where the rays converge.
  const char *env = getenv("EI_K1_SMEM_KB");
  Chunks ch1, chRS;
  int RC4 = 0, RS = 1, cps = 2, ntile = 0;
  long long ctas = 0;
  std::vector<int> rf_flags;
  size_t budget = 0;
  auto plan_rs = [&](int rt) {
    p.proj.RT = rt;
    cps = rt == RT ? 2 : 4;   // CTAs per SM
    budget = (env ? (size_t)atoi(env) : (cps == 2 ? 104 : 50)) * 1024;
    const size_t budget4 = (cps == 2 ? 100 : 50) * 1024;
    int rc = 32;
    for (;;) {   // rows per chunk of a 4-stage ring at the widest window (sets the row split)
      Chunks t;
      build_chunks(p, angles, groups, order, 1, 1 << 30, rc, t);
      if ((size_t)NSTMAX * rc * (t.wmax + 2) * per_entry <= budget4 || rc == 1) break;
      rc /= 2;
    }
    RC4 = rc;
    ntile = (ND + rt - 1) / rt;
    ctas = (long long)ntile * (long long)groups.size() * p.S;
    // row split for small problems: the largest power of two keeping the grid within one wave
    // of cps CTAs per SM (measured best on C2 with 64-ray tiles: RS = 2)
    RS = 1;
    while (RS < 8 && ctas * RS * 2 <= (long long)cps * sms && N / (RS * 2) >= 2 * RC4) RS *= 2;
    if (const char *e = getenv("EI_K1_RS")) RS = std::max(1, std::min(8, atoi(e)));   // tuning knob
  };
  {   // per angle group, the lane mapping with fewer modelled shared-memory wavefronts, stored in
      // bit 16 of the group's count (tuning knob EI_K1_RAYFAST forces one mapping everywhere)
    const char *force = getenv("EI_K1_RAYFAST");
    rf_flags.assign(groups.size(), 0);
    double wa_sum = 0.0, wbest = 0.0;
    int nrf = 0;
    for (size_t g = 0; g < groups.size(); ++g) {
      const double wa = wavefront_model(p, angles, groups, order, g, false);
      const double wr = wavefront_model(p, angles, groups, order, g, true);
      int rf = wr < 0.9 * wa ? 1 : 0;
      if (force) rf = atoi(force) ? 1 : 0;
      wa_sum += wa;
      wbest += rf ? wr : wa;
      nrf += rf;
      rf_flags[g] = rf;   // encoded into the device copy at the end (host code reads counts)
    }
    p.proj.ray_fast = nrf;
    if (getenv("EI_PLAN_VERBOSE"))
      fprintf(stderr, "libei plan: K1 modelled wavefronts/sample angle-fast %.2f chosen %.2f (%d/%d ray-fast groups)\n",
              wa_sum / groups.size(), wbest / groups.size(), nrf, (int)groups.size());
  }  // Ray tile: 64 rays; 32 when the 64-ray grid is one wave on more CTAs than SMs (C2, P1): twice
  // the units at four CTAs per SM balance the heavy and light units of the wave better (C2 K1
  // 39.2 -> 34.8 us; multi-wave grids keep 64: C4 K1 8.65 vs 9.13 ms with 32, C5 1.23 vs 1.49).
  plan_rs(RT);
  const long long grid64 = ctas * RS;
  int rt_use = (grid64 > sms && grid64 <= 2LL * sms) ? RTS : RT;
  // also for dense views whose 64-ray windows only allow small chunks (C3: K1 0.620 -> 0.603 ms);
  // not for sparse views, where 32-ray tiles add bank conflicts (C5: 1.23 -> 1.49 ms)
  if (RC4 <= 4 && 4 * p.proj.ray_fast < (int)groups.size()) rt_use = RTS;
  if (const char *e = getenv("EI_K1_RT")) rt_use = atoi(e) == RTS ? RTS : RT;   // tuning knob
  if (rt_use != RT) plan_rs(rt_use);
  // K0 triggers K1's launch at its start only for grids smaller than the SMs (C1: 28.8 -> 26.8
  // us): a larger single-wave grid launched while K0 occupies SMs would not land as the unit
  // placement below assumes (C2 with 32-ray tiles: 73.4 -> 79.3 us)
  p.proj.k0_early = ctas * RS <= sms ? 1 : 0;
  if (const char *e = getenv("EI_K0_EARLY")) p.proj.k0_early = atoi(e) ? 1 : 0;   // tuning knob
  int nst = 2;
  int RCMAX = 1;
  while (RCMAX * 2 <= std::max(1, (N / RS) / 2) && RCMAX < 32) RCMAX *= 2;
  if (const char *e = getenv("EI_K1_RC")) RCMAX = std::max(1, atoi(e));   // tuning knob: rows per chunk cap
  auto stage_entries = [&](int n) { return (int)(budget / ((size_t)n * per_entry)) & ~1; };
  if (!build_chunks(p, angles, groups, order, 1, stage_entries(nst), RCMAX, ch1)) return EI_ERR_SHAPE;
  // 32-ray tiles: a third stage where it fits the 4-CTA budget (C2 72.0 -> 71.6 us, P1 39.2 -> 38.9)
  if (p.proj.RT == RTS && (size_t)3 * ch1.rcmax * (ch1.wmax + 2) * per_entry <= budget) nst = 3;
  if (const char *e = getenv("EI_K1_NST")) nst = std::max(2, std::min(NSTMAX, atoi(e)));   // knob
  const int E = stage_entries(nst);
  if (!build_chunks(p, angles, groups, order, 1, E, RCMAX, ch1)) return EI_ERR_SHAPE;
  // K1B band mode for the cost / forward path of small maps: units (group, band of BR = 16 map
  // rows, slice) of nearly equal work, every lane sweeping all N_d rays.  Measured
  // (tools/dbg/sweep_band.sh, step time): P1 (N_d = N) 38.8 -> 37.0 us (378 units); C2 (N_d = 1.5 N:
  // a third of the lanes sample zero entries) 68.2 -> 87 us with 384 units, 81 us at BR = 11 (576
  // units, K2 summing 24 partials); C1 (N_d = 1.5 N, 48 units) 26.7 -> 26.8-27.5 us.  So: BR = 16
  // rows fit the 104 KB budget, N_d <= 1.2 N, and the band grid within 1.5 waves of 2 CTAs per SM
  // (knobs EI_K1_BAND, EI_K1_BR)
  p.proj.band = 0;
  {
    const int bstride = (N + 4 + 1) & ~1;
    const int brmax = std::min(64, (int)((size_t)104 * 1024 / ((size_t)bstride * per_entry)));
    const int br0 = 16;
    const long long units16 = (long long)((N + br0 - 1) / br0) * (long long)groups.size() * p.S;
    bool use = brmax >= br0 && 5LL * ND <= 6LL * N && units16 <= 3LL * sms && 2 * units16 >= sms;
    int br = br0;
    if (const char *e = getenv("EI_K1_BAND")) use = atoi(e) != 0 && brmax >= 4;
    if (const char *e = getenv("EI_K1_BR")) br = atoi(e);
    br = std::max(1, std::min(brmax, br));
    const int nb = (N + br - 1) / br;
    if (use && (size_t)nb * p.S * 3 * NA * ND * sizeof(float) <= ((size_t)256 << 20)) {
      p.proj.band = 1;
      p.proj.BR = br;
      p.proj.bstride = bstride;
      RS = nb;
      p.proj.k0_early = (long long)nb * groups.size() * p.S <= sms ? 1 : 0;
    }
  }
  if (p.proj.band) {
    chRS = ch1;
  } else if (RS > 1) {
    if (!build_chunks(p, angles, groups, order, RS, E, RCMAX, chRS)) return EI_ERR_SHAPE;
  } else {
    chRS = ch1;
  }
  if (k1_smem(nst, E, std::max(ch1.nchmax, chRS.nchmax), 3) > 220 * 1024) return EI_ERR_SHAPE;
  if (getenv("EI_PLAN_VERBOSE"))
    fprintf(stderr, "libei plan: K1 RT %d angles %d RS %d nst %d E %d: %zu chunks, <= %d per unit, %.2f rows avg, <= %d rows, "
            "widest window %d\n", p.proj.RT, 4 * p.proj.nsl, RS, nst, E, ch1.c.size(), ch1.nchmax,
            ch1.c.empty() ? 0.0 : (double)[&] { long long r = 0; for (auto &q : ch1.c) r += q.w; return r; }() / ch1.c.size(),
            ch1.rcmax, ch1.wmax);
  if (getenv("EI_PLAN_VERBOSE") && p.proj.band)
    fprintf(stderr, "libei plan: K1B band mode: %d bands of %d rows x %zu groups x %d slices (stride %d)\n",
            RS, p.proj.BR, groups.size(), p.S, p.proj.bstride);
  p.proj.E = E;
  p.proj.nst = nst;
  p.proj.n_groups = (int)groups.size();
  p.proj.RS = RS;
  p.proj.nchmax1 = ch1.nchmax;
  p.proj.nchmaxRS = chRS.nchmax;
  p.proj.rcmax = std::max(ch1.rcmax, chRS.rcmax);
  p.proj.wmax = std::max(ch1.wmax, chRS.wmax);
  // zero padding of the pair-layout map rows so every staged window is one in-bounds copy
  p.proj.PAD = ((p.proj.wmax + 1) & ~1) + 2;   // even
  p.proj.Rp = (N + 1 + 2 * p.proj.PAD + 1) & ~1;   // even: 16-B aligned float2 rows
  p.proj.n_tiles = ntile;
  if ((long long)ntile * groups.size() * p.S * RS > 0x7fffffffLL) return EI_ERR_SHAPE;   // 1-D grid
  unit1 = order_units(ch1, 1, (int)groups.size(), ntile, p.S, cps);
  unitRS = (RS > 1 && !p.proj.band) ? order_units(chRS, RS, (int)groups.size(), ntile, p.S, cps) : unit1;
  chunks1.swap(ch1.c);
  coff1.swap(ch1.off);
  if (RS > 1 && !p.proj.band) {
    chunksRS.swap(chRS.c);
    coffRS.swap(chRS.off);
  } else {
    chunksRS.clear();
    coffRS.clear();
  }
  for (size_t g = 0; g < groups.size(); ++g) groups[g].y |= rf_flags[g] << 16;   // last: device copy
  return EI_OK;
}

cudaError_t launch_project3(const ei_plan &p, float *P, int RS, cudaStream_t st) {
  return launch<3>(p, RS, P, st);
}

cudaError_t launch_project1(const ei_plan &p, float *P, cudaStream_t st, int RS) {
  return launch<1>(p, RS, P, st);
}

}  // namespace ei

#ifdef EI_TRACE
extern "C" int ei_debug_k1_trace(unsigned long long *host, int n_ctas) {
  n_ctas = n_ctas < 65536 ? n_ctas : 65536;
  return cudaMemcpyFromSymbol(host, ei::g_k1_trace, sizeof(unsigned long long) * 4 * n_ctas) == cudaSuccess ? 0 : 5;
}
#endif

#ifdef EI_TRACE
extern "C" int ei_debug_span_proj(unsigned long long *host, int reset) {
  if (reset) {
    unsigned long long init[8];
    for (int k = 0; k < 4; ++k) { init[2 * k] = ~0ULL; init[2 * k + 1] = 0ULL; }
    return cudaMemcpyToSymbol(ei::g_span_proj, init, sizeof(init)) == cudaSuccess ? 0 : 5;
  }
  return cudaMemcpyFromSymbol(host, ei::g_span_proj, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 5;
}
#endif
