// k_backproject.cu — K3: the adjoint R^T as a pixel-driven, atomic-free tent gather
// ("exact algebraic transpose").  For pixel (i, j) and
// angle theta the Joseph weight of ray k is (dx/|c_dom|) max(0, 1 - |k - k*|/h) with
// k* = (x_j cos + y_i sin)/du + (Nd-1)/2 and h = |c_dom| dx/du <= 1, so only the detector pair
// (floor(k*), floor(k*)+1) contributes (du >= dx is enforced by the plan).
//
// B200 design:
//  * gradient sinograms arrive in a PAIR layout written by K2: entry e of a row holds
//    (g[e-1], g[e]) for every map, so one tap pair of all three maps is one LDS.128 + one LDS.64
//    (A = (mu0, mu1, delta0, delta1), B = (sigma0, sigma1)); row length Nd+1 (e = 0..Nd).
//  * a CTA owns a 32x32 pixel tile (256 consumer threads x 4 pixels) and walks the angles in
//    chunks of 16; a producer warp stages, per angle, only the 48-entry detector window the tile
//    projects onto, with 1-D bulk copies (TMA engine) into a 3-stage shared-memory ring that
//    completes on full/empty mbarriers (G rows are zero-padded, so every window is one
//    in-bounds copy); consumer warps never meet a CTA-wide barrier in the loop;
//  * a warp covers an 8x4 pixel sub-tile, whose taps fall on ~10 consecutive window entries:
//    lanes share (broadcast) most loads, ~3 shared-memory wavefronts per 32 pixel-angles;
//  * the pair products accumulate with FFMA2 (__ffma2_rn: two fp32 FMAs per instruction on
//    sm_100a): acc.x collects the left taps, acc.y the right taps, summed once at the end.
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

template <int NMAP>
struct Layout;
template <>
struct Layout<3> {   // A = (mu0, mu1, delta0, delta1), B = (sigma0, sigma1)
  using A = float4;
  static constexpr bool hasB = true;
};
template <>
struct Layout<1> {   // A = (g0, g1)
  using A = float2;
  static constexpr bool hasB = false;
};

// staged windows: separate planes (16-B and 8-B element strides keep the LDS.128 / LDS.64 of a
// quarter/half warp on distinct banks; an interleaved 32-B entry stride measured 1.5x slower)
template <int NMAP>
struct Smem {
  typename Layout<NMAP>::A a[NST][CH][sizeof(typename Layout<NMAP>::A) == 8 ? WLB : WL];
  float2 b[NST][CH][Layout<NMAP>::hasB ? WLB : 2];
  float4 tab[NST][CH];
  int ws[NST][CH];
  uint64_t full[NST], empty[NST];
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

template <int NMAP, bool TAB>
__global__ void __launch_bounds__(NT + 32, 3) backproject_kernel(
    const typename Layout<NMAP>::A *__restrict__ GA, const float2 *__restrict__ GB,
    const float4 *__restrict__ k3, const int *__restrict__ alist, int NA3, int N, int NA, int ND,
    const float *__restrict__ mu,
    const float *__restrict__ delta, const float *__restrict__ sigma, float lambda,
    float *__restrict__ o0, float *__restrict__ o1, float *__restrict__ o2, size_t out_stride,
    int S, int KS, float *__restrict__ part3, int PADG, int RpG,
    const int4 *__restrict__ units, FinArgs fin) {
  using TA = typename Layout<NMAP>::A;
  constexpr bool A8 = sizeof(TA) == 8;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem<NMAP> &sm = *reinterpret_cast<Smem<NMAP> *>(smem_raw);
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
  const TA *GAs = GA + (size_t)s * NA * rowlen + PADG;
  const float2 *GBs = GB ? GB + (size_t)s * NA * rowlen + PADG : nullptr;
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
    pdl_wait();   // K2's gradient sinograms
    // tile corners (full 32x32 tile, even past the map edge, so every lane indexes the window)
    const float xa = (float)j0 - ctr, xb = xa + (float)(TILE - 1);
    const float ya = (float)i0 - ctr, yb = ya + (float)(TILE - 1);
    const uint32_t bytesA = A8 ? (uint32_t)WLB * 8 : (uint32_t)WL * 16;
    const uint32_t bytesB = NMAP == 3 ? (uint32_t)WLB * 8 : 0u;
    int st = 0;
    uint32_t ph = 0;
    for (int c = c_lo; c < c_hi; ++c) {
      if (c - c_lo >= NST) mbar_wait(&sm.empty[st], ph ^ 1);
      const int na = min(CH, a_hi - a_lo - c * CH);
      int ws = 0;
      if (lane < na) {   // per-angle table + window start (first tap entry - 1)
        const int a = __ldg(alist_k + c * CH + lane);
        const float4 g = __ldg(k3 + a);   // cdu, sdu, inv_h, scale
        const float k00 = fmaf(xa, g.x, fmaf(ya, g.y, dctr)), k01 = fmaf(xb, g.x, fmaf(ya, g.y, dctr));
        const float k10 = fmaf(xa, g.x, fmaf(yb, g.y, dctr)), k11 = fmaf(xb, g.x, fmaf(yb, g.y, dctr));
        ws = (int)floorf(fminf(fminf(k00, k01), fminf(k10, k11))) - 1;
        sm.tab[st][lane] = make_float4(g.x, g.y, g.z, 1.f - g.z);   // cdu, sdu, 1/h, 1 - 1/h
        sm.ws[st][lane] = ws;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], (uint32_t)na * (bytesA + bytesB));
      __syncwarp();
      if (lane < na) {
        const size_t row = (size_t)__ldg(alist_k + c * CH + lane) * rowlen;
        // a window entirely off the detector only needs zeros: clamp its copy into the zero pad
        // (a window overlapping [0, ND] is always inside the PADG >= WL padding)
        const int e0 = min(max(ws + 1, -PADG), ND + PADG - WLB), eb = e0 & ~1;
        bulk_g2s(&sm.a[st][lane][0], GAs + row + (A8 ? eb : e0), bytesA, &sm.full[st]);
        if (NMAP == 3) bulk_g2s(&sm.b[st][lane][0], GBs + row + eb, bytesB, &sm.full[st]);
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

  float2 am[4], ad[4], as[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) am[q] = ad[q] = as[q] = make_float2(0.f, 0.f);

  pdl_wait();   // sleep while K2 runs (this CTA may have launched early)
  int st = 0;
  uint32_t ph = 0;
  for (int c = c_lo; c < c_hi; ++c) {
    mbar_wait(&sm.full[st], ph);
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
      const TA *arow = &sm.a[st][al][A8 ? bofs : 0];
      const float2 *brow = &sm.b[st][Layout<NMAP>::hasB ? al : 0][bofs];
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
        const TA ga = arow[k0];
        if constexpr (NMAP == 3) {
          am[q] = __ffma2_rn(wt, make_float2(ga.x, ga.y), am[q]);
          ad[q] = __ffma2_rn(wt, make_float2(ga.z, ga.w), ad[q]);
          as[q] = __ffma2_rn(wt, brow[k0], as[q]);
        } else {
          am[q] = __ffma2_rn(wt, ga, am[q]);
        }
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
        float *pp = part3 + ((size_t)(ks * S + s) * 3) * NN + (size_t)i * N + j;
        pp[0] = am[q].x + am[q].y;
        if constexpr (NMAP == 3) {
          pp[NN] = ad[q].x + ad[q].y;
          pp[2 * NN] = as[q].x + as[q].y;
        }
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
    if constexpr (NMAP == 3) {
      float vd = ad[q].x + ad[q].y, vs = as[q].x + as[q].y;
      if (mu) {   // cost path: + 2 lambda x (eq. 5); maps have slice stride N*N
        const size_t ip = (size_t)s * NN + p;
        const float l2 = 2.f * lambda;
        vm = fmaf(l2, __ldg(mu + ip), vm);
        vd = fmaf(l2, __ldg(delta + ip), vd);
        vs = fmaf(l2, __ldg(sigma + ip), vs);
      }
      o0[oo] = vm;
      o1[oo] = vd;
      o2[oo] = vs;
    } else {
      if (mu) vm = fmaf(2.f * lambda, __ldg(mu + (size_t)s * NN + p), vm);   // single-map cost path
      o0[oo] = vm;
    }
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

template <int NMAP>
cudaError_t launch_bp(const ei_plan &p, const typename Layout<NMAP>::A *GA, const float2 *GB,
                      const float *mu, const float *delta, const float *sigma, float lambda,
                      float *o0, float *o1, float *o2, size_t out_stride, const Finalize *fz,
                      cudaStream_t st) {
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
  const size_t smem = sizeof(Smem<NMAP>);
  cudaError_t e = cudaFuncSetAttribute((const void *)backproject_kernel<NMAP, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute((const void *)backproject_kernel<NMAP, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid = p.k3u ? dim3(p.n_k3u) : dim3((p.N + TILE - 1) / TILE, (p.N + TILE - 1) / TILE, p.S * p.KS);
  auto kern = p.k3u ? backproject_kernel<NMAP, true> : backproject_kernel<NMAP, false>;
  e = launch_pdl(kern, grid, dim3(NT + 32), smem, st, GA, GB, p.tab.k3, p.alist3,
                 p.NA3, p.N, p.NA, p.ND, mu, delta, sigma, lambda, o0, o1, o2, out_stride, p.S, p.KS, p.part3,
                 p.PADG, p.RpG, (const int4 *)p.k3u, fin);
  if (e != cudaSuccess) return e;
  if (p.KS > 1) {
    const size_t total = (size_t)p.S * p.N * p.N;
    const int blocks = (int)std::min<size_t>((total + 255) / 256, 148 * 8);
    e = launch_pdl(ks_reduce_kernel<NMAP>, dim3(blocks), dim3(256), 0, st, (const float *)p.part3, p.KSk,
                   p.KSe, p.S, p.N, mu, delta, sigma, lambda, o0, o1, o2, out_stride);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace

int bp_pad() { return 64; }   // G row padding (entries) >= window width WL + slack, even
int bp_tiles(int N) { return ((N + TILE - 1) / TILE) * ((N + TILE - 1) / TILE); }
int bp_chunks(int NA) { return (NA + CH - 1) / CH; }

cudaError_t launch_backproject3(const ei_plan &p, const float *mu, const float *delta,
                                const float *sigma, float lambda, float *g_mu, float *g_delta,
                                float *g_sigma, size_t out_stride, const Finalize *fin,
                                cudaStream_t st) {
  return launch_bp<3>(p, p.GA, p.GB, mu, delta, sigma, lambda, g_mu, g_delta, g_sigma, out_stride, fin,
                      st);
}

cudaError_t launch_backproject1(const ei_plan &p, float *map, cudaStream_t st, const float *h,
                                float lambda, const Finalize *fin) {
  return launch_bp<1>(p, p.GA1, nullptr, h, nullptr, nullptr, lambda, map, nullptr, nullptr,
                      (size_t)p.N * p.N, fin, st);
}

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
