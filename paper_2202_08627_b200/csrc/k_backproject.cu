// k_backproject.cu — K3: the adjoint R^T as a pixel-driven, atomic-free tent gather
// ("exact algebraic transpose").  For pixel (i, j) and
// angle theta the Joseph weight of ray k is (dx/|c_dom|) max(0, 1 - |k - k*|/h) with
// k* = (x_j cos + y_i sin)/du + (Nd-1)/2 and h = |c_dom| dx/du <= 1, so only the detector pair
// (floor(k*), floor(k*)+1) contributes (du >= dx is enforced by the plan).
//
// B200 design — three-map model (backproject3_kernel), bound by the shared-memory data pipe:
//  * gradient sinograms arrive in a TRIPLE layout written by K2: entry e of a row holds the three
//    detector values e-1, e, e+1 of every map in three planes, A = (m[e-1], m[e], s[e-1], s[e]),
//    B = (d[e-1], d[e], m[e+1], d[e+1]), C = s[e+1] (m, d, s = the mu, delta, sigma gradients
//    pre-scaled by the Joseph weight), e = -1..Nd, zero outside the detector;
//  * a thread owns horizontally adjacent PIXEL PAIRS: their k* differ by |c'| = |cos| dx/du <= 1,
//    so the pair's four taps lie in three consecutive detector positions and one entry serves both
//    pixels — 36 B (LDS.128 + LDS.128 + LDS.32) per pixel pair instead of 24 B per pixel (the pair
//    layout's LDS.128 + LDS.64), i.e. 4.5 instead of >= 6 shared-memory wavefronts per 32 pixels;
//    the lower pixel (smaller k*) takes the tent weights of its two taps, the upper one three tent
//    weights over the entry's three positions (max(0, 1 - |k - k*|/h), identical values);
//  * which pixel of a pair is lower depends on the sign of cos(theta) only: the plan lists the
//    back-projected angles cos >= 0 first, and the per-pixel partial sums of the first class are
//    folded into totals at the (warp-uniform) class change;
//  * a CTA owns a 32x32 pixel tile (256 consumer threads x 2 pairs; a quarter warp = 4 pair columns
//    x 2 rows, whose entries span <= 8 consecutive entries: no bank conflicts) and walks the angles
//    in chunks of 16; a producer warp stages, per angle, the 48-entry detector window of the tile
//    (1-D bulk copies, TMA engine) into a 2-stage mbarrier ring;
//  * FFMA2 (two fp32 FMAs per instruction on sm_100a) on the taps held in aligned register pairs.
// Single-map model (backproject1_kernel): the PAIR layout (g[e-1], g[e]) per entry, one LDS.64 per
// pixel, a 3-stage ring, warp = 8x4 pixel sub-tile with 4 pixels per thread.
// Nothing is scattered: deterministic.  The cost path adds 2*lambda*x (eq. 5).
#include <algorithm>

#include "ei_common.cuh"
#include "tma.cuh"

namespace ei {
namespace {

#ifdef EI_TRACE
// debug builds only (tools/dbg/step_trace.py): earliest CTA start / latest CTA end of this file's
// kernels in the last traced call (globaltimer, ns)
__device__ unsigned long long g_span_bp[2 * 4];
__device__ __forceinline__ unsigned long long gt_bp() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SPAN_START_bp() const unsigned long long span_t0_ = gt_bp()
#define SPAN_END_bp(k)                                   \
  do {                                                    \
    atomicMin(&g_span_bp[2 * (k)], span_t0_);            \
    atomicMax(&g_span_bp[2 * (k) + 1], gt_bp());         \
  } while (0)
#else
#define SPAN_START_bp()
#define SPAN_END_bp(k)
#endif

constexpr int TILE = 32;   // pixels per side
constexpr int CH = 16;     // angles per staged chunk
constexpr int WL = 48;     // window entries per angle (>= 31*sqrt(2) + 4)
constexpr int NT = 256;     // consumer threads (+ one producer warp)
constexpr int NST = 3;      // ring stages
constexpr int WLB = WL + 2; // 8-byte-entry rows: 16-B aligned copy start needs one spare entry

// single-map staged windows (pair layout, 8-B entries)
struct Smem1 {
  float2 a[NST][CH][WLB];
  float4 tab[NST][CH];
  int ws[NST][CH];
  uint64_t full[NST], empty[NST];
};

// three-map staged windows (triple layout): planes of 16-B, 16-B and 4-B entries (separate planes
// keep each LDS on distinct banks), all starting at the same entry e0, a multiple of 4 (16-B aligned
// C-plane copies), so one index addresses all three; e0 <= floor(min k*) + 1 - 0 and the window
// holds WL3 = 52 >= 45 + 4 entries
#ifndef EI_K3_NST3
#define EI_K3_NST3 2
#endif
#ifndef EI_K3_CH3
#define EI_K3_CH3 16
#endif
constexpr int NST3 = EI_K3_NST3;   // ring stages (compile-time switches for A/B runs)
constexpr int CH3 = EI_K3_CH3;     // angles per staged chunk
constexpr int WL3 = 52;
// one staged angle: its three planes and its table in one record, so a single pointer (stepped
// once per angle) addresses everything the consumers read for it (immediate offsets)
struct Ang3 {
  float4 a[WL3];   // (m[e-1], m[e], s[e-1], s[e])
  float4 b[WL3];   // (d[e-1], d[e], m[e+1], d[e+1])
  float c[WL3];    // s[e+1]
  float4 t1;       // c', s', 1/h, 1 - 1/h
  float4 t2;       // (Nd-1)/2 + 1 - e0 + min(c', 0), |c'| - 1, -, -
};
struct Smem3 {
  Ang3 ang[NST3][CH3];
  int nb[NST3];              // first angle of the chunk with cos < 0 (CH if none)
  float tot[12][NT];        // per consumer thread: totals of finished angle classes (pair, L/R, map)
  uint64_t full[NST3], empty[NST3];
};

#ifdef EI_TRACE
// debug builds only (tools/dbg/k1_trace.py --k3): per CTA {start, first chunk staged, end, SM id}
__device__ unsigned long long g_k3_trace[4 * 65536];
__device__ __forceinline__ unsigned long long gtimer3() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

struct FinArgs {
  const double *part_cost;            // K2 per-warp partials [S][NA][nseg * nw]
  const float *part_mo;
  const double *part_reg;
  int per_slice, nseg, NA, RB;   // per_slice = NA * nseg * nw, nseg here = nseg * nw
  double lambda;
  double *cost;                  // NULL: no finalize (ei_backproject)
  float *g_drift;                // [S][NA] or NULL
  int *diag;                     // -DEI_CHECK builds: staged-window overflows (ei_plan_info out[4])
};

// consumer threads only (named barrier 1, NT threads); fixed order: per-thread strided fp64 sums,
// then the warps' sums in warp order
__device__ __forceinline__ void finalize(const FinArgs &f, int s, int tid) {
  __shared__ double fred[NT / 32];
  // every thread's loads are issued UF at a time (independent L2 round trips in flight) and added
  // in the same strided order as a plain loop: q = tid, tid + NT, ...
  constexpr int UF = 8;
  double c = 0.0, rg = 0.0;
  const double *pc = f.part_cost + (size_t)s * f.per_slice;
  int q = tid;
  for (; q + (UF - 1) * NT < f.per_slice; q += UF * NT) {
    double v[UF];
#pragma unroll
    for (int u = 0; u < UF; ++u) v[u] = __ldcg(pc + q + u * NT);
#pragma unroll
    for (int u = 0; u < UF; ++u) c += v[u];
  }
  for (; q < f.per_slice; q += NT) c += __ldcg(pc + q);
  if (f.lambda > 0.0)
    for (int b = tid; b < f.RB; b += NT) rg += __ldcg(f.part_reg + (size_t)s * f.RB + b);
  double v = c + f.lambda * rg;
  for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
  if ((tid & 31) == 0) fred[tid >> 5] = v;
  asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < NT / 32; ++w) t += fred[w];
    f.cost[s] = t;
  }
  if (f.g_drift)
    for (int a = tid; a < f.NA; a += NT) {
      const float *pm = f.part_mo + ((size_t)s * f.NA + a) * f.nseg;
      double m = 0.0;
      int r = 0;
      for (; r + UF <= f.nseg; r += UF) {
        float v[UF];
#pragma unroll
        for (int u = 0; u < UF; ++u) v[u] = __ldcg(pm + r + u);
#pragma unroll
        for (int u = 0; u < UF; ++u) m += (double)v[u];
      }
      for (; r < f.nseg; ++r) m += (double)__ldcg(pm + r);
      f.g_drift[(size_t)s * f.NA + a] = (float)m;
    }
}

// single-map model (NEXT-3): pair layout (g[e-1], g[e]) per entry
template <bool TAB>
__global__ void __launch_bounds__(NT + 32, 3) backproject1_kernel(
    const float2 *__restrict__ GA, const float4 *__restrict__ k3, const int *__restrict__ alist,
    int NA3, int N, int NA, int ND, const float *__restrict__ mu, float lambda,
    float *__restrict__ o0, size_t out_stride,
    int S, int KS, float *__restrict__ part3, int PADG, int RpG,
    const int4 *__restrict__ units, FinArgs fin) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem1 &sm = *reinterpret_cast<Smem1 *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // unit: tile, slice, part ks of the tile's angle split into nks parts.  Grids with more units
  // than SMs read it from the plan's placement table (parts of unequal size placed heaviest first);
  // the others decode it from the block index, grid (tiles x, tiles y, KS x S), with no table load
  // ahead of the first copy
  int j0, i0, s, ks, nks;
  if (TAB) {   // (separate instantiation: the untabled kernel keeps its own code schedule)
    const int4 u = __ldg(units + blockIdx.x);
    const int ntx = (N + TILE - 1) / TILE;
    j0 = (u.x % ntx) * TILE; i0 = (u.x / ntx) * TILE; s = u.y; ks = u.z; nks = u.w;
  } else {
    j0 = blockIdx.x * TILE; i0 = blockIdx.y * TILE; s = blockIdx.z % S; ks = blockIdx.z / S; nks = KS;
  }
SPAN_START_bp();
#ifdef EI_TRACE
  const unsigned long long t_start = gtimer3();
  unsigned long long t_data = 0;
#endif
  const float ctr = 0.5f * (float)(N - 1), dctr = 0.5f * (float)(ND - 1);
  const size_t rowlen = (size_t)RpG;   // padded G rows: entry e at e + PADG
  const float2 *GAs = GA + (size_t)s * NA * rowlen + PADG;
  // angle split (small grids): CTA ks owns angles [a_lo, a_hi) of the back-projected list, an equal
  // share (not a whole number of chunks: 360 angles in 6 parts are 60 each, staged as 16+16+16+12,
  // where whole chunks gave 3 or 4 chunks per CTA), in chunks of CH staged angles
  const int a_lo = (int)(((long long)ks * NA3) / nks), a_hi = (int)(((long long)(ks + 1) * NA3) / nks);
  const int c_lo = 0, c_hi = (a_hi - a_lo + CH - 1) / CH;
  const int *alist_k = alist + a_lo;

  if (tid == 0) {
    for (int q = 0; q < NST; ++q) {
      mbar_init(&sm.full[q], 1);
      mbar_init(&sm.empty[q], NT / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // PDL: the producer (TMA of K2's gradient rows) and the finalize CTAs (K2's partials) wait for
  // K2; the other consumers only read what the producer staged
  if (w == NT / 32) {   // ---------------- producer warp ----------------
    // the first chunk's tables (plan data) are prepared before the PDL wait, see backproject3
    // tile corners (full 32x32 tile, even past the map edge, so every lane indexes the window)
    const float xa = (float)j0 - ctr, xb = xa + (float)(TILE - 1);
    const float ya = (float)i0 - ctr, yb = ya + (float)(TILE - 1);
    const uint32_t bytesA = (uint32_t)WLB * 8;
    int st = 0;
    uint32_t ph = 0;
    for (int c = c_lo; c < c_hi; ++c) {
      if (c - c_lo >= NST) mbar_wait(&sm.empty[st], ph ^ 1);
      const int na = min(CH, a_hi - a_lo - c * CH);
      int ws = 0, a = 0;
      if (lane < na) {   // per-angle table + window start (first tap entry - 1)
        a = __ldg(alist_k + c * CH + lane);
        const float4 g = __ldg(k3 + a);   // cdu, sdu, inv_h, scale
        const float k00 = fmaf(xa, g.x, fmaf(ya, g.y, dctr)), k01 = fmaf(xb, g.x, fmaf(ya, g.y, dctr));
        const float k10 = fmaf(xa, g.x, fmaf(yb, g.y, dctr)), k11 = fmaf(xb, g.x, fmaf(yb, g.y, dctr));
        ws = (int)floorf(fminf(fminf(k00, k01), fminf(k10, k11))) - 1;
        sm.tab[st][lane] = make_float4(g.x, g.y, g.z, 1.f - g.z);   // cdu, sdu, 1/h, 1 - 1/h
        sm.ws[st][lane] = ws;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], (uint32_t)na * bytesA);
      __syncwarp();
      if (c == c_lo) pdl_wait();   // K2's gradient sinograms
      if (lane < na) {
        const size_t row = (size_t)a * rowlen;
        // a window entirely off the detector only needs zeros: clamp its copy into the zero pad
        // (a window overlapping [0, ND] is always inside the PADG >= WL padding)
        const int e0 = min(max(ws + 1, -PADG), ND + PADG - WLB), eb = e0 & ~1;
        bulk_g2s(&sm.a[st][lane][0], GAs + row + eb, bytesA, &sm.full[st]);
      }
      if (++st == NST) { st = 0; ph ^= 1; }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  // fused K4 (cost path): while the producer fills the ring, CTA (0, 0, s) of angle split 0 sums
  // K2's per-segment partials of slice s in index order (+ lambda * K0's sum x^2 partials) and
  // the per-angle drift gradient
  if (fin.cost && i0 == 0 && j0 == 0 && ks == 0) {
    pdl_wait();   // K2's partials
    finalize(fin, s, tid);
  }
  const int row = 4 * w + (lane >> 3), lx = lane & 7;
  const float yi = (float)(i0 + row) - ctr;
  float xq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) xq[q] = (float)(j0 + lx + 8 * q) - ctr;

  float2 am[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) am[q] = make_float2(0.f, 0.f);

  pdl_wait();   // sleep while K2 runs (this CTA may have launched early)
  int st = 0;
  uint32_t ph = 0;
  for (int c = c_lo; c < c_hi; ++c) {
    mbar_wait_full(&sm.full[st], ph);
#ifdef EI_TRACE
    if (c == c_lo) t_data = gtimer3();
#endif
    const int na = min(CH, a_hi - a_lo - c * CH);
#pragma unroll 2   // two angles in flight per warp (measured: C4 K3 8.94 -> 8.76 ms; x4 8.80)
    for (int al = 0; al < na; ++al) {
      const float4 t = sm.tab[st][al];
      const int ws = sm.ws[st][al];
      const int bofs = (ws + 1) & 1;
      const float base = fmaf(yi, t.y, dctr - (float)ws);
      const float2 *arow = &sm.a[st][al][bofs];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float kst = fmaf(xq[q], t.x, base);   // window-local k*, > 0
        const int k0 = __float2int_rd(kst);
        const float fr = kst - (float)k0;
        // tent weights of the pair (k0, k0+1); G was pre-scaled by dx/|c_dom| in K2, so each
        // weight is one saturating FMA: max(0, 1 - |k - k*|/h) with |k - k*|/h <= 1/h
        const float2 wt = make_float2(__saturatef(fmaf(-fr, t.z, 1.f)), __saturatef(fmaf(fr, t.z, t.w)));
#ifdef EI_CHECK
        // debug build: the pair (k0, k0+1) lies inside the staged window of WL entries
        if (k0 < 0 || k0 + 1 >= WL) atomicAdd(fin.diag, 1);
#endif
        am[q] = __ffma2_rn(wt, arow[k0], am[q]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);
    if (++st == NST) { st = 0; ph ^= 1; }
  }

#ifdef EI_TRACE
  asm volatile("bar.sync 2, %0;\n" ::"n"(NT) : "memory");   // consumers only
  if (tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const size_t b = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;   // linear
    if (b < 65536) {
      g_k3_trace[4 * b] = t_start;
      g_k3_trace[4 * b + 1] = t_data;
      g_k3_trace[4 * b + 2] = gtimer3();
      g_k3_trace[4 * b + 3] = smid | ((unsigned long long)(c_hi - c_lo) << 32);
    }
    SPAN_END_bp(0);
  }
#endif
  const int i = i0 + row;
  const size_t NN = (size_t)N * N;
  if (KS > 1) {   // angle split: publish partials; ks_reduce_kernel sums them in part order
    if (i < N) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + lx + 8 * q;
        if (j >= N) continue;
        part3[((size_t)(ks * S + s) * 3) * NN + (size_t)i * N + j] = am[q].x + am[q].y;
      }
    }
    return;
  }
  if (i >= N) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = j0 + lx + 8 * q;
    if (j >= N) continue;
    const size_t p = (size_t)i * N + j;
    const size_t oo = (size_t)s * out_stride + p;
    float vm = am[q].x + am[q].y;
    if (mu) vm = fmaf(2.f * lambda, __ldg(mu + (size_t)s * NN + p), vm);   // cost path: + 2 lambda h
    o0[oo] = vm;
  }
}

// three-map model: triple layout, pixel pairs (see the file header)
template <bool TAB>
__global__ void __launch_bounds__(NT + 32, 3) backproject3_kernel(
    const float4 *__restrict__ GA, const float4 *__restrict__ GB, const float *__restrict__ GC,
    const float4 *__restrict__ k3, const int *__restrict__ alist, int NA3, int N, int NA, int ND,
    const float *__restrict__ mu, const float *__restrict__ delta, const float *__restrict__ sigma,
    float lambda, float *__restrict__ o0, float *__restrict__ o1, float *__restrict__ o2,
    size_t out_stride, int S, int KS, float *__restrict__ part3, int PADG, int RpG,
    const int4 *__restrict__ units, FinArgs fin) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem3 &sm = *reinterpret_cast<Smem3 *>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int j0, i0, s, ks, nks;   // unit decode as in backproject1_kernel
  if (TAB) {
    const int4 u = __ldg(units + blockIdx.x);
    const int ntx = (N + TILE - 1) / TILE;
    j0 = (u.x % ntx) * TILE; i0 = (u.x / ntx) * TILE; s = u.y; ks = u.z; nks = u.w;
  } else {
    j0 = blockIdx.x * TILE; i0 = blockIdx.y * TILE; s = blockIdx.z % S; ks = blockIdx.z / S; nks = KS;
  }
SPAN_START_bp();
#ifdef EI_TRACE
  const unsigned long long t_start = gtimer3();
  unsigned long long t_data = 0;
#endif
  const float ctr = 0.5f * (float)(N - 1), dctr = 0.5f * (float)(ND - 1);
  const size_t rowlen = (size_t)RpG, soff = (size_t)s * NA * rowlen + PADG;
  const int a_lo = (int)(((long long)ks * NA3) / nks), a_hi = (int)(((long long)(ks + 1) * NA3) / nks);
#ifndef EI_K3_CH0
#define EI_K3_CH0 8
#endif
  // chunk c holds angles [c0(c), c0(c) + na(c)): a first chunk of CH0 = 8 <= CH angles lets the
  // consumers start before a whole chunk has landed (C4 K3 8.13 -> 8.07 ms, C1 15.0 -> 13.7 us;
  // 4 angles: the same on C4, slower on C1; compile-time switch EI_K3_CH0)
  constexpr int CH0 = EI_K3_CH0;
  const int nang = a_hi - a_lo;
  const int c_hi = nang <= CH0 ? 1 : 1 + (nang - CH0 + CH3 - 1) / CH3;
  auto c0 = [&](int c) { return c == 0 ? 0 : CH0 + (c - 1) * CH3; };
  auto nac = [&](int c) { return min(c == 0 ? CH0 : CH3, nang - c0(c)); };
  const int *alist_k = alist + a_lo;

  if (tid == 0) {
    for (int q = 0; q < NST3; ++q) {
      mbar_init(&sm.full[q], 1);
      mbar_init(&sm.empty[q], NT / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (w == NT / 32) {   // ---------------- producer warp ----------------
    // the per-angle tables and windows are plan data: the first chunk's are prepared before the
    // PDL wait (they overlap K2's tail); only the copies of K2's gradient rows wait for K2
    const float xa = (float)j0 - ctr, xb = xa + (float)(TILE - 1);
    const float ya = (float)i0 - ctr, yb = ya + (float)(TILE - 1);
    constexpr uint32_t bytesAB = (uint32_t)WL3 * 16, bytesC = (uint32_t)WL3 * 4;
    int st = 0;
    uint32_t ph = 0;
    for (int c = 0; c < c_hi; ++c) {
      if (c >= NST3) mbar_wait(&sm.empty[st], ph ^ 1);
      const int na = nac(c);
      int e0 = 0, a = 0;
      if (lane < na) {   // per-angle tables + window start
        a = __ldg(alist_k + c0(c) + lane);
        const float4 g = __ldg(k3 + a);   // c', s', 1/h, Joseph weight
        const float k00 = fmaf(xa, g.x, fmaf(ya, g.y, dctr)), k01 = fmaf(xb, g.x, fmaf(ya, g.y, dctr));
        const float k10 = fmaf(xa, g.x, fmaf(yb, g.y, dctr)), k11 = fmaf(xb, g.x, fmaf(yb, g.y, dctr));
        // first entry the tile needs (floor of the smallest k*, + 1), one of slack, rounded down
        // to a multiple of 4; a window entirely off the detector only needs zeros: clamp its copy
        // into the zero pad (a window overlapping [-1, ND] is never clamped: PADG >= WL3 + 8)
        const int ws = (int)floorf(fminf(fminf(k00, k01), fminf(k10, k11))) - 1;
        e0 = min(max((ws + 1) & ~3, -PADG + 4), (RpG - PADG - WL3 - 4) & ~3);
        sm.ang[st][lane].t1 = make_float4(g.x, g.y, g.z, 1.f - g.z);
        sm.ang[st][lane].t2 = make_float4(dctr + 1.f - (float)e0 + fminf(g.x, 0.f), fabsf(g.x) - 1.f, 0.f, 0.f);
      }
      {   // first angle of the chunk with cos < 0 (the list has cos >= 0 first), na if none
        const unsigned neg = __ballot_sync(0xffffffffu, lane < na && sm.ang[st][lane].t1.x < 0.f);
        if (lane == 0) sm.nb[st] = neg ? __ffs(neg) - 1 : na;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], (uint32_t)na * (2u * bytesAB + bytesC));
      __syncwarp();
      if (c == 0) pdl_wait();   // K2's gradient sinograms
      if (lane < na) {
        const size_t row = soff + (size_t)a * rowlen + e0;
        bulk_g2s(&sm.ang[st][lane].a[0], GA + row, bytesAB, &sm.full[st]);
        bulk_g2s(&sm.ang[st][lane].b[0], GB + row, bytesAB, &sm.full[st]);
        bulk_g2s(&sm.ang[st][lane].c[0], GC + row, bytesC, &sm.full[st]);
      }
      if (++st == NST3) { st = 0; ph ^= 1; }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  if (fin.cost && i0 == 0 && j0 == 0 && ks == 0) {   // fused K4 (see backproject1_kernel)
    pdl_wait();
    finalize(fin, s, tid);
  }
  // warp w covers a 16 x 8 pixel block (2 x 4 blocks per tile); lane = (pair column pc, row r):
  // a quarter warp is 4 pair columns x 2 rows; pair p of a thread sits 8 pixels right of pair 0
  const int wx = w & 1, wy = w >> 1, pc = lane & 3, r = lane >> 2;
  const int row = 8 * wy + r, jl = j0 + 16 * wx + 2 * pc;      // left pixel of pair 0
  const float yi = (float)(i0 + row) - ctr;
  const float xl0 = (float)jl - ctr, xl1 = xl0 + 8.f;
  // partial sums of the current class: lower pixel (2 taps: float2 per map), upper pixel (3 taps:
  // float2 + float per map); totals of finished classes per (pair, left/right, map)
  float2 lm0 = make_float2(0.f, 0.f), ld0 = lm0, ls0 = lm0, hm0 = lm0, hd0 = lm0, hs0 = lm0;
  float2 lm1 = lm0, ld1 = lm0, ls1 = lm0, hm1 = lm0, hd1 = lm0, hs1 = lm0;
  float2 hmd30 = lm0, hmd31 = lm0;   // upper pixel's third tap of mu and delta: one FFMA2 (u2 broadcast)
  float2 hs3p = lm0;                 // and of sigma, pair 0 in .x, pair 1 in .y (one FFMA2 per angle)
  // totals of finished classes in shared memory (this thread's column; touched once per class):
  // tot[(2 p + side) 3 + map][tid], side 0 = left pixel
#pragma unroll
  for (int m = 0; m < 12; ++m) sm.tot[m][tid] = 0.f;
  int cls = 0;   // 0: cos >= 0, lower pixel = left; 1: cos < 0, lower pixel = right
  auto flush = [&]() {   // fold the class's partial sums into the per-pixel totals, restart
    const float L[2][3] = {{lm0.x + lm0.y, ld0.x + ld0.y, ls0.x + ls0.y},
                           {lm1.x + lm1.y, ld1.x + ld1.y, ls1.x + ls1.y}};
    const float H[2][3] = {{hm0.x + hm0.y + hmd30.x, hd0.x + hd0.y + hmd30.y, hs0.x + hs0.y + hs3p.x},
                           {hm1.x + hm1.y + hmd31.x, hd1.x + hd1.y + hmd31.y, hs1.x + hs1.y + hs3p.y}};
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        sm.tot[(2 * p) * 3 + m][tid] += cls ? H[p][m] : L[p][m];
        sm.tot[(2 * p + 1) * 3 + m][tid] += cls ? L[p][m] : H[p][m];
      }
    lm0 = ld0 = ls0 = hm0 = hd0 = hs0 = lm1 = ld1 = ls1 = hm1 = hd1 = hs1 = make_float2(0.f, 0.f);
    hmd30 = hmd31 = hs3p = make_float2(0.f, 0.f);
  };

  pdl_wait();   // sleep while K2 runs (this CTA may have launched early)
  int st = 0;
  uint32_t ph = 0;
  for (int c = 0; c < c_hi; ++c) {
    mbar_wait_full(&sm.full[st], ph);
#ifdef EI_TRACE
    if (c == 0) t_data = gtimer3();
#endif
    const int na = nac(c);
    // the chunk's angles of the current class, then (at most once per CTA) the class change
    // and the rest: the plan lists cos >= 0 first, so the change is one index per chunk
    const int nb = cls ? na : min(na, sm.nb[st]);
    auto angle = [&](const Ang3 *ap) {   // the loop runs on this pointer
      const float4 t1 = ap->t1, t2 = ap->t2;
      const float4 *ar = ap->a, *br = ap->b;
      const float *cr = ap->c;
      const float base = fmaf(yi, t1.y, t2.x);   // staged index of the lower pixel's entry, - x term
      auto pair = [&](float xl, float2 &lm, float2 &ld, float2 &ls, float2 &hm, float2 &hd, float2 &hs,
                      float2 &hmd3, float &u2o, float &Co) {
        const float kst = fmaf(xl, t1.x, base);   // lower pixel's k* + 1 - e0 (> 0)
        const int k0 = __float2int_rd(kst);
        const float fr = kst - (float)k0;
        // lower pixel: taps k0, k0+1; upper pixel (k* + |c'|, |c'| <= 1): taps k0, k0+1, k0+2 with
        // the tent max(0, 1 - |k - k*|/h) at distances f1, |f1 - 1|, 2 - f1, written with
        // x = f1 - 1 in [-1, 1): 1 - (1 + x)/h, 1 - |x|/h, 1 - (1 - x)/h (one FFMA.SAT each)
        const float2 wl = make_float2(__saturatef(fmaf(-fr, t1.z, 1.f)), __saturatef(fmaf(fr, t1.z, t1.w)));
        const float x1 = fr + t2.y;
        const float2 u01 = make_float2(__saturatef(fmaf(-x1, t1.z, t1.w)), __saturatef(fmaf(-fabsf(x1), t1.z, 1.f)));
        const float u2 = __saturatef(fmaf(x1, t1.z, t1.w));
#ifdef EI_CHECK
        if (k0 < 0 || k0 >= WL3) atomicAdd(fin.diag, 1);   // debug build: inside the staged window
#endif
        const float4 A = ar[k0], B = br[k0];
        const float C = cr[k0];
        lm = __ffma2_rn(wl, make_float2(A.x, A.y), lm);
        ls = __ffma2_rn(wl, make_float2(A.z, A.w), ls);
        ld = __ffma2_rn(wl, make_float2(B.x, B.y), ld);
        hm = __ffma2_rn(u01, make_float2(A.x, A.y), hm);
        hs = __ffma2_rn(u01, make_float2(A.z, A.w), hs);
        hd = __ffma2_rn(u01, make_float2(B.x, B.y), hd);
        hmd3 = __ffma2_rn(make_float2(u2, u2), make_float2(B.z, B.w), hmd3);   // FFMA2, scalar operand
        u2o = u2;
        Co = C;
      };
      float u20, u21, C0, C1;
      pair(xl0, lm0, ld0, ls0, hm0, hd0, hs0, hmd30, u20, C0);
      pair(xl1, lm1, ld1, ls1, hm1, hd1, hs1, hmd31, u21, C1);
      hs3p = __ffma2_rn(make_float2(u20, u21), make_float2(C0, C1), hs3p);   // both pairs' sigma third taps
    };
    const Ang3 *a0 = &sm.ang[st][0];
#pragma unroll 1
    for (const Ang3 *ap = a0; ap != a0 + nb; ++ap) angle(ap);
    if (nb < na) {   // the class changes inside this chunk (warp-uniform)
      flush();
      cls = 1;
#pragma unroll 1
      for (const Ang3 *ap = a0 + nb; ap != a0 + na; ++ap) angle(ap);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);
    if (++st == NST3) { st = 0; ph ^= 1; }
  }
  flush();
#ifdef EI_TRACE
  asm volatile("bar.sync 2, %0;\n" ::"n"(NT) : "memory");   // consumers only
  if (tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const size_t b = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;   // linear
    if (b < 65536) {
      g_k3_trace[4 * b] = t_start;
      g_k3_trace[4 * b + 1] = t_data;
      g_k3_trace[4 * b + 2] = gtimer3();
      g_k3_trace[4 * b + 3] = smid | ((unsigned long long)c_hi << 32);
    }
    SPAN_END_bp(0);
  }
#endif
  const int i = i0 + row;
  if (i >= N) return;
  const size_t NN = (size_t)N * N;
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int j = jl + 8 * p + q;
      if (j >= N) continue;
      const size_t px = (size_t)i * N + j;
      float v0 = sm.tot[(2 * p + q) * 3][tid], v1 = sm.tot[(2 * p + q) * 3 + 1][tid],
            v2 = sm.tot[(2 * p + q) * 3 + 2][tid];
      if (KS > 1) {   // angle split: publish partials; ks_reduce_kernel sums them in part order
        float *pp = part3 + ((size_t)(ks * S + s) * 3) * NN + px;
        pp[0] = v0;
        pp[NN] = v1;
        pp[2 * NN] = v2;
        continue;
      }
      if (mu) {   // cost path: + 2 lambda x (eq. 5); maps have slice stride N*N
        const size_t ip = (size_t)s * NN + px;
        const float l2 = 2.f * lambda;
        v0 = fmaf(l2, __ldg(mu + ip), v0);
        v1 = fmaf(l2, __ldg(delta + ip), v1);
        v2 = fmaf(l2, __ldg(sigma + ip), v2);
      }
      const size_t oo = (size_t)s * out_stride + px;
      o0[oo] = v0;
      o1[oo] = v1;
      o2[oo] = v2;
    }
}

// angle split (KS > 1): fixed-order sum of the KS partial gradients + 2 lambda x (eq. 5), one thread
// per (slice, pixel), launched with PDL right after K3
template <int NMAP>
__global__ void __launch_bounds__(256) ks_reduce_kernel(const float *__restrict__ part3, int KSk, int KSe, int S,
                                                        int N, const float *__restrict__ mu,
                                                        const float *__restrict__ delta,
                                                        const float *__restrict__ sigma, float lambda,
                                                        float *__restrict__ o0, float *__restrict__ o1,
                                                        float *__restrict__ o2, size_t out_stride) {
  SPAN_START_bp();
  pdl_wait();
  const size_t NN = (size_t)N * N, total = (size_t)S * NN;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const size_t s = t / NN, p = t - s * NN;
    int KS = KSk;
    if (KSe > 0) {   // the first KSe (slice, tile) pairs have one part more
      const int ntx = (N + TILE - 1) / TILE, tile = (int)(p / N) / TILE * ntx + (int)(p % N) / TILE;
      KS += (long long)s * ntx * ntx + tile < KSe ? 1 : 0;
    }
    float v[3] = {0.f, 0.f, 0.f};
    for (int k2 = 0; k2 < KS; ++k2) {
      const float *pp = part3 + ((size_t)(k2 * S + s) * 3) * NN + p;
#pragma unroll
      for (int m = 0; m < (NMAP == 3 ? 3 : 1); ++m) v[m] += __ldcg(pp + m * NN);
    }
    const size_t oo = s * out_stride + p;
    if (mu) {
      const float l2 = 2.f * lambda;
      v[0] = fmaf(l2, __ldg(mu + s * NN + p), v[0]);
      if (NMAP == 3) {
        v[1] = fmaf(l2, __ldg(delta + s * NN + p), v[1]);
        v[2] = fmaf(l2, __ldg(sigma + s * NN + p), v[2]);
      }
    }
    o0[oo] = v[0];
    if (NMAP == 3) {
      o1[oo] = v[1];
      o2[oo] = v[2];
    }
  }
  pdl_trigger();
#ifdef EI_TRACE
  __syncthreads();
  if (threadIdx.x == 0) SPAN_END_bp(1);
#endif
}

FinArgs fin_args(const ei_plan &p, float lambda, const Finalize *fz) {
  FinArgs fin{};
  fin.diag = p.diag;
  if (fz) {
    fin.part_cost = p.part_curve;
    fin.part_mo = p.part_mo;
    fin.part_reg = p.part_reg;
    fin.per_slice = p.NA * p.k2.nseg * p.k2.nw;
    fin.nseg = p.k2.nseg * p.k2.nw;
    fin.NA = p.NA;
    fin.RB = p.RB;
    fin.lambda = (double)lambda;
    fin.cost = fz->cost;
    fin.g_drift = fz->g_drift;
  }
  return fin;
}

template <class K>
cudaError_t set_smem(K kt, K kf, size_t smem) {
  cudaError_t e = cudaFuncSetAttribute((const void *)kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void *)kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return e;
}

dim3 bp_grid(const ei_plan &p) {
  return p.k3u ? dim3(p.n_k3u) : dim3((p.N + TILE - 1) / TILE, (p.N + TILE - 1) / TILE, p.S * p.KS);
}

template <int NMAP>
cudaError_t launch_ks_reduce(const ei_plan &p, const float *mu, const float *delta, const float *sigma,
                             float lambda, float *o0, float *o1, float *o2, size_t out_stride,
                             cudaStream_t st) {
  if (p.KS <= 1) return cudaSuccess;
  const size_t total = (size_t)p.S * p.N * p.N;
  const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 8);
  return launch_pdl(ks_reduce_kernel<NMAP>, dim3(blocks), dim3(256), 0, st, (const float *)p.part3, p.KSk,
                    p.KSe, p.S, p.N, mu, delta, sigma, lambda, o0, o1, o2, out_stride);
}

}  // namespace

cudaError_t launch_backproject3(const ei_plan &p, const float *mu, const float *delta,
                                const float *sigma, float lambda, float *g_mu, float *g_delta,
                                float *g_sigma, size_t out_stride, const Finalize *fz,
                                cudaStream_t st) {
  const FinArgs fin = fin_args(p, lambda, fz);
  cudaError_t e = set_smem(backproject3_kernel<true>, backproject3_kernel<false>, sizeof(Smem3));
  if (e != cudaSuccess) return e;
  auto kern = p.k3u ? backproject3_kernel<true> : backproject3_kernel<false>;
  e = launch_pdl(kern, bp_grid(p), dim3(NT + 32), sizeof(Smem3), st, (const float4 *)p.GA,
                 (const float4 *)p.GB, (const float *)p.GC, p.tab.k3, p.alist3, p.NA3, p.N, p.NA, p.ND, mu,
                 delta, sigma, lambda, g_mu, g_delta, g_sigma, out_stride, p.S, p.KS, p.part3, p.PADG,
                 p.RpG, (const int4 *)p.k3u, fin);
  if (e == cudaSuccess)
    e = launch_ks_reduce<3>(p, mu, delta, sigma, lambda, g_mu, g_delta, g_sigma, out_stride, st);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t launch_backproject1(const ei_plan &p, float *map, cudaStream_t st, const float *h,
                                float lambda, const Finalize *fz) {
  const FinArgs fin = fin_args(p, lambda, fz);
  cudaError_t e = set_smem(backproject1_kernel<true>, backproject1_kernel<false>, sizeof(Smem1));
  if (e != cudaSuccess) return e;
  const size_t os = (size_t)p.N * p.N;
  auto kern = p.k3u ? backproject1_kernel<true> : backproject1_kernel<false>;
  e = launch_pdl(kern, bp_grid(p), dim3(NT + 32), sizeof(Smem1), st, (const float2 *)p.GA1, p.tab.k3,
                 p.alist3, p.NA3, p.N, p.NA, p.ND, h, lambda, map, os, p.S, p.KS, p.part3, p.PADG, p.RpG,
                 (const int4 *)p.k3u, fin);
  if (e == cudaSuccess)
    e = launch_ks_reduce<1>(p, h, nullptr, nullptr, lambda, map, nullptr, nullptr, os, st);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

int bp_pad() { return 64; }   // G row padding (entries) >= window width WL3 + 12, multiple of 4
int bp_tiles(int N) { return ((N + TILE - 1) / TILE) * ((N + TILE - 1) / TILE); }
int bp_chunks(int NA) { return (NA + CH - 1) / CH; }

}  // namespace ei

#ifdef EI_TRACE
extern "C" int ei_debug_k3_trace(unsigned long long *host, int n_ctas) {
  n_ctas = n_ctas < 65536 ? n_ctas : 65536;
  return cudaMemcpyFromSymbol(host, ei::g_k3_trace, sizeof(unsigned long long) * 4 * n_ctas) == cudaSuccess ? 0 : 5;
}
#endif

#ifdef EI_TRACE
extern "C" int ei_debug_span_bp(unsigned long long *host, int reset) {
  if (reset) {
    unsigned long long init[8];
    for (int k = 0; k < 4; ++k) { init[2 * k] = ~0ULL; init[2 * k + 1] = 0ULL; }
    return cudaMemcpyToSymbol(ei::g_span_bp, init, sizeof(init)) == cudaSuccess ? 0 : 5;
  }
  return cudaMemcpyFromSymbol(host, ei::g_span_bp, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 5;
}
#endif
