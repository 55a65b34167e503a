// k_pack.cu — K0: re-layout the maps for the projector.
//
// PAIR layout: the Joseph sample at x* needs (x[j0], x[j0+1]) with j0 = floor(x*).  K0 writes,
// for every map row, N+1 entries where entry e = (x[e-1], x[e]) (zero outside the row), so the
// projector fetches the tap pair of all three maps with one 16-B + one 8-B shared-memory load:
//   MA[e] = (mu[e-1], mu[e], delta[e-1], delta[e]),  MB[e] = (sigma[e-1], sigma[e]).
// The same is written for the TRANSPOSED maps (rows = columns): column-dominant angles are
// projected as row-dominant angles of the transposed map with (cos, sin) swapped (hard part H2),
// so the projector only ever walks contiguous rows.
// K0 also counts non-finite map elements into status[0] and emits per-tile sum(x^2) partials for
// the eq. 5 regulariser.
#include <algorithm>

#include "ei_common.cuh"
#include "tma.cuh"

namespace ei {
namespace {

#ifdef EI_TRACE
// debug builds only (tools/dbg/step_trace.py): earliest CTA start / latest CTA end of this file's
// kernels in the last traced call (globaltimer, ns)
__device__ unsigned long long g_span_pack[2 * 4];
__device__ __forceinline__ unsigned long long gt_pack() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SPAN_START_pack() const unsigned long long span_t0_ = gt_pack()
#define SPAN_END_pack(k)                                   \
  do {                                                    \
    atomicMin(&g_span_pack[2 * (k)], span_t0_);            \
    atomicMax(&g_span_pack[2 * (k) + 1], gt_pack());         \
  } while (0)
#else
#define SPAN_START_pack()
#define SPAN_END_pack(k)
#endif

constexpr int T = 16;

template <int NMAP>
struct PairOut;
template <>
struct PairOut<3> {
  float4 *a, *aT;
  float2 *b, *bT;
};
template <>
struct PairOut<1> {
  float2 *a, *aT;
};

// grid (ceil((N+1)/T), ceil((N+1)/T), S), block (T, T), T = 16.  Tile (ta, tb) loads map rows
// [T ta - 1, T ta + T - 1] x cols [T tb - 1, T tb + T - 1] and writes normal entries (rows T ta..,
// entries T tb..) and transposed entries (T-rows T tb.., entries T ta..).
template <int NMAP>
__global__ void __launch_bounds__(256) pack_pairs_kernel(const float *__restrict__ in0,
                                                         const float *__restrict__ in1,
                                                         const float *__restrict__ in2,
                                                         size_t in_stride, int N, PairOut<NMAP> out,
                                                         double *__restrict__ part_reg,
                                                         int32_t *__restrict__ status,
                                                         SmallCheck chk, int nflat, int M, int NA,
                                                         int PAD, int Rp, int trigger_early) {
  __shared__ float tile[NMAP][T + 1][T + 2];   // (T+1)^2 with a one-element halo
  __shared__ double red[8];
  SPAN_START_pack();
  // small K1 grids (fewer CTAs than SMs): let K1's CTAs launch now (they wait for this grid before
  // reading its output); larger single-wave K1 grids are placed by the plan assuming an empty GPU,
  // so they launch when this grid completes (plan_projector)
  if (trigger_early) PDL_TRIGGER_K0();
  const int s = blockIdx.z, ta = blockIdx.y, tb = blockIdx.x;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * T + tx;
  const float *src[3] = {in0 + s * in_stride, NMAP == 3 ? in1 + s * in_stride : nullptr,
                         NMAP == 3 ? in2 + s * in_stride : nullptr};
  double sq = 0.0;
  int bad = 0;
  // load (T+1) x (T+1) with a one-element halo above and to the left
  for (int q = tid; q < (T + 1) * (T + 1); q += T * T) {
    const int r = q / (T + 1), c = q - r * (T + 1);
    const int i = ta * T - 1 + r, j = tb * T - 1 + c;
    const bool in = (i >= 0 && i < N && j >= 0 && j < N);
#pragma unroll
    for (int m = 0; m < NMAP; ++m) {
      const float v = in ? __ldg(src[m] + (size_t)i * N + j) : 0.f;
      tile[m][r][c] = v;
      if (in && r >= 1 && c >= 1) {   // owned pixel: count once
        bad += !isfinite(v);
        sq += (double)v * v;
      }
    }
  }
  __syncthreads();
  const size_t rl = (size_t)Rp, slice = (size_t)N * rl;   // entry e stored at e + PAD
  // normal: row i = T ta + r, entry e = T tb + c -> (x[i][e-1], x[i][e]) = tile[r+1][c], tile[r+1][c+1]
  // transposed: T-row j = T tb + r, entry e = T ta + c -> (x[e-1][j], x[e][j]) = tile[c][r+1], tile[c+1][r+1]
  {
    const int r = ty, c = tx;
    const int i = ta * T + r, e = tb * T + c;
    if (i < N && e <= N) {
      const size_t o = s * slice + (size_t)i * rl + PAD + e;
      if constexpr (NMAP == 3) {
        out.a[o] = make_float4(tile[0][r + 1][c], tile[0][r + 1][c + 1], tile[1][r + 1][c], tile[1][r + 1][c + 1]);
        out.b[o] = make_float2(tile[2][r + 1][c], tile[2][r + 1][c + 1]);
      } else {
        out.a[o] = make_float2(tile[0][r + 1][c], tile[0][r + 1][c + 1]);
      }
    }
    const int j = tb * T + r, eT = ta * T + c;
    if (j < N && eT <= N) {
      const size_t o = s * slice + (size_t)j * rl + PAD + eT;
      if constexpr (NMAP == 3) {
        out.aT[o] = make_float4(tile[0][c][r + 1], tile[0][c + 1][r + 1], tile[1][c][r + 1], tile[1][c + 1][r + 1]);
        out.bT[o] = make_float2(tile[2][c][r + 1], tile[2][c + 1][r + 1]);
      } else {
        out.aT[o] = make_float2(tile[0][c][r + 1], tile[0][c + 1][r + 1]);
      }
    }
  }
  if (status && chk.flat) {   // this CTA's share of the flat/mask/drift non-finite scan
    const int total = nflat + M + (chk.drift ? NA : 0);
    const int nb = gridDim.x * gridDim.y * gridDim.z;
    const int b = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const int per = (total + nb - 1) / nb;
    for (int t = b * per + tid; t < min(total, (b + 1) * per); t += T * T) {
      const float v = t < nflat ? chk.flat[t] : (t < nflat + M ? chk.mask[t - nflat] : chk.drift[t - nflat - M]);
      bad += !isfinite(v);
    }
  }
  if (status && bad) atomicAdd(&status[0], bad);   // integer count: order-independent
  if (part_reg) {
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, off);
    if ((tid & 31) == 0) red[tid >> 5] = sq;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      part_reg[(size_t)s * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
  }
#ifdef EI_TRACE
  __syncthreads();
  if (tid == 0) SPAN_END_pack(0);
#endif
}

// planar sino [S][NMAP][NA][ND] -> pair layout [S][NA][ND+1] (entry e = (g[e-1], g[e]))
// (each value pre-multiplied by the angle's Joseph weight dx/|c_dom|, as K2 does)
// ei_backproject's input sinograms -> K3's layout, pre-multiplied by the Joseph weight: three
// maps the TRIPLE layout (entries e = -1..ND: positions e-1, e, e+1 of every map, see
// ei_common.cuh), one map the PAIR layout (entries e = 0..ND: (g[e-1], g[e])).  One thread per
// (slice, angle, entry).
template <int NMAP>
__global__ void pack_sino_kernel(const float *__restrict__ in, int NA, int ND, int S,
                                 float4 *__restrict__ GA, float4 *__restrict__ GB,
                                 float *__restrict__ GC, float2 *__restrict__ GA1,
                                 const float4 *__restrict__ k3, int PADG, int RpG) {
  const size_t plane = (size_t)NA * ND, rl = (size_t)ND + 2;   // entries -1..ND
  const size_t total = (size_t)S * NA * rl;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t sa = t / rl;
    const int e = (int)(t - sa * rl) - 1;
    const size_t o = sa * (size_t)RpG + PADG + e;
    const size_t s = sa / NA, a = sa - s * NA;
    const float *b = in + s * NMAP * plane + a * ND;
    const float sc = __ldg(k3 + a).w;
    auto at = [&](int m, int k) { return (k >= 0 && k < ND) ? sc * __ldg(b + m * plane + k) : 0.f; };
    if (NMAP == 3) {
      GA[o] = make_float4(at(0, e - 1), at(0, e), at(2, e - 1), at(2, e));
      GB[o] = make_float4(at(1, e - 1), at(1, e), at(0, e + 1), at(1, e + 1));
      GC[o] = at(2, e + 1);
    } else if (e >= 0) {
      GA1[o] = make_float2(at(0, e - 1), at(0, e));
    }
  }
}


// Mirror-pair fold (360-degree scans): the angle theta + pi sees the same lines as theta with the
// detector mirrored, k -> ND-1-k (R6), so R^T g = sum over primaries of R_theta^T (g_theta +
// mirror(g_{theta+pi})).  In place on the primary rows (a); the partner's (b) value at position k
// is the centre of its entry k: g_b(k) = m: GA.y, d: GB.y, s: GA.w (three maps).  Three maps,
// entry e (positions e-1, e, e+1) gains g_b at ND-e, ND-1-e, ND-2-e; one map, entry e (positions
// e-1, e) gains the partner's entry ND-e with its two taps swapped.  Partner entries outside -1..ND lie in the zero
// padding.  One thread per (slice, pair, entry).
template <int NMAP>
__global__ void __launch_bounds__(256) fold_kernel(const int2 *__restrict__ pairs, int npairs, int NA,
                                                   int ND, int S, float4 *__restrict__ GA,
                                                   float4 *__restrict__ GB, float *__restrict__ GC,
                                                   float2 *__restrict__ GA1, int PADG, int RpG) {
  pdl_wait();   // K2's (or pack_sino's) gradient rows
  const long long rl = ND + 2, total = (long long)S * npairs * rl;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int e = (int)(t % rl) - 1;
    const long long sp = t / rl;
    const int q = (int)(sp % npairs), s = (int)(sp / npairs);
    const int2 ab = __ldg(pairs + q);
    const size_t oa = ((size_t)s * NA + ab.x) * RpG + PADG + e;
    const size_t ob = ((size_t)s * NA + ab.y) * RpG + PADG;   // partner row, entry 0
    if (NMAP == 3) {
      const float4 b0 = GA[ob + ND - e], b1 = GA[ob + ND - 1 - e], b2 = GA[ob + ND - 2 - e];
      const float4 c0 = GB[ob + ND - e], c1 = GB[ob + ND - 1 - e], c2 = GB[ob + ND - 2 - e];
      const float4 x = GA[oa], y = GB[oa];
      GA[oa] = make_float4(x.x + b0.y, x.y + b1.y, x.z + b0.w, x.w + b1.w);
      GB[oa] = make_float4(y.x + c0.y, y.y + c1.y, y.z + b2.y, y.w + c2.y);
      GC[oa] += b2.w;
    } else if (e >= 0) {   // partner entry ND-e = (g_b(ND-e-1), g_b(ND-e)), taps swapped
      const float2 u = GA1[oa], v = GA1[ob + ND - e];
      GA1[oa] = make_float2(u.x + v.y, u.y + v.x);
    }
  }
  pdl_trigger();
}

}  // namespace

cudaError_t launch_fold(const ei_plan &p, int n_maps, cudaStream_t st) {
  if (p.npairs == 0) return cudaSuccess;
  const long long total = (long long)p.S * p.npairs * (p.ND + 2);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  if (n_maps == 3)
    return launch_pdl(fold_kernel<3>, dim3(blocks), dim3(256), 0, st, (const int2 *)p.pairs, p.npairs,
                      p.NA, p.ND, p.S, p.GA, p.GB, p.GC, (float2 *)nullptr, p.PADG, p.RpG);
  return launch_pdl(fold_kernel<1>, dim3(blocks), dim3(256), 0, st, (const int2 *)p.pairs, p.npairs,
                    p.NA, p.ND, p.S, (float4 *)nullptr, (float4 *)nullptr, (float *)nullptr, p.GA1, p.PADG,
                    p.RpG);
}

int reg_blocks(int N) { return ((N + 1 + T - 1) / T) * ((N + 1 + T - 1) / T); }

cudaError_t launch_pack3(const ei_plan &p, const float *mu, const float *delta, const float *sigma,
                         size_t in_stride, bool want_reg, int32_t *status, SmallCheck chk,
                         cudaStream_t st) {
  const int nt = (p.N + 1 + T - 1) / T;
  dim3 grid(nt, nt, p.S), block(T, T);
  PairOut<3> o{p.MA, p.MAT, p.MB, p.MBT};
  pack_pairs_kernel<3><<<grid, block, 0, st>>>(mu, delta, sigma, in_stride, p.N, o,
                                               want_reg ? p.part_reg : nullptr, status, chk,
                                               p.S * (chk.nflat_per_slice ? chk.nflat_per_slice : 3 * p.ND),
                                               chk.mask ? p.M : 0, p.NA, p.proj.PAD, p.proj.Rp,
                                               p.proj.k0_early);
  return cudaGetLastError();
}

cudaError_t launch_pack1(const ei_plan &p, const float *map, cudaStream_t st, bool want_reg,
                         int32_t *status, SmallCheck chk) {
  const int nt = (p.N + 1 + T - 1) / T;
  dim3 grid(nt, nt, p.S), block(T, T);
  PairOut<1> o{p.M1, p.M1T};
  pack_pairs_kernel<1><<<grid, block, 0, st>>>(map, nullptr, nullptr, (size_t)p.N * p.N, p.N, o,
                                               want_reg ? p.part_reg : nullptr, status, chk,
                                               p.S * (chk.nflat_per_slice ? chk.nflat_per_slice : 3 * p.ND),
                                               chk.mask ? p.M : 0, p.NA, p.proj.PAD, p.proj.Rp,
                                               p.proj.k0_early);
  return cudaGetLastError();
}

cudaError_t launch_pack_sino(const ei_plan &p, const float *sino, int n_maps, cudaStream_t st) {
  const size_t total = (size_t)p.S * p.NA * (p.ND + 2);
  const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  if (n_maps == 3)
    pack_sino_kernel<3><<<blocks, 256, 0, st>>>(sino, p.NA, p.ND, p.S, p.GA, p.GB, p.GC, nullptr,
                                                p.tab.k3, p.PADG, p.RpG);
  else
    pack_sino_kernel<1><<<blocks, 256, 0, st>>>(sino, p.NA, p.ND, p.S, nullptr, nullptr, nullptr, p.GA1,
                                                p.tab.k3, p.PADG, p.RpG);
  return cudaGetLastError();
}


}  // namespace ei

#ifdef EI_TRACE
extern "C" int ei_debug_span_pack(unsigned long long *host, int reset) {
  if (reset) {
    unsigned long long init[8];
    for (int k = 0; k < 4; ++k) { init[2 * k] = ~0ULL; init[2 * k + 1] = 0ULL; }
    return cudaMemcpyToSymbol(ei::g_span_pack, init, sizeof(init)) == cudaSuccess ? 0 : 5;
  }
  return cudaMemcpyFromSymbol(host, ei::g_span_pack, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 5;
}
#endif
