// k_backproject.cu — K3: the adjoint R^T as a pixel-driven, atomic-free tent gather
// ("exact algebraic transpose").  For pixel (i, j) and
// angle theta the Joseph weight of ray k is (dx/|c_dom|) max(0, 1 - |k - k*|/h) with
// k* = (x_j cos + y_i sin)/du + (Nd-1)/2 and h = |c_dom| dx/du <= 1, so at most the two
// detector taps floor(k*) and floor(k*)+1 contribute (du >= dx is enforced by the plan).
// One thread = one pixel; it loops over all angles; nothing is scattered, so the result is
// deterministic.  The cost path adds the eq. 5 regulariser gradient 2 lambda x here.
#include "ei_common.cuh"

namespace ei {
namespace {

constexpr int BX = 32, BY = 8;

template <int NMAP>
struct GT;
template <>
struct GT<3> {
  using T = float4;
};
template <>
struct GT<1> {
  using T = float;
};

__device__ __forceinline__ void fma_acc(float4 &acc, float w, float4 g) {
  acc.x = fmaf(w, g.x, acc.x);
  acc.y = fmaf(w, g.y, acc.y);
  acc.z = fmaf(w, g.z, acc.z);
}
__device__ __forceinline__ void fma_acc(float &acc, float w, float g) { acc = fmaf(w, g, acc); }

template <int NMAP>
__global__ void __launch_bounds__(BX *BY) backproject_kernel(
    const typename GT<NMAP>::T *__restrict__ G, const float4 *__restrict__ k3, int N, int NA,
    int ND, const float *__restrict__ mu, const float *__restrict__ delta,
    const float *__restrict__ sigma, float lambda, float *__restrict__ o0, float *__restrict__ o1,
    float *__restrict__ o2, size_t out_stride) {
  using T = typename GT<NMAP>::T;
  extern __shared__ float4 stab[];   // [NA] angle table
  for (int a = threadIdx.y * BX + threadIdx.x; a < NA; a += BX * BY) stab[a] = __ldg(k3 + a);
  __syncthreads();
  const int j = blockIdx.x * BX + threadIdx.x, i = blockIdx.y * BY + threadIdx.y;
  const int s = blockIdx.z;
  if (i >= N || j >= N) return;
  const float ctr = 0.5f * (float)(N - 1), dctr = 0.5f * (float)(ND - 1);
  const float xj = (float)j - ctr, yi = (float)i - ctr;
  const T *Gs = G + (size_t)s * NA * ND;
  T acc;
  if constexpr (NMAP == 3) acc = make_float4(0.f, 0.f, 0.f, 0.f); else acc = 0.f;
  for (int a = 0; a < NA; ++a) {
    const float4 t = stab[a];   // cdu, sdu, inv_h, scale
    const float ks = fmaf(xj, t.x, fmaf(yi, t.y, dctr));
    const float f = floorf(ks);
    const int k0 = (int)f;
    const float fr = ks - f;
    const float w0 = fmaxf(0.f, fmaf(-fr, t.z, 1.f)) * t.w;
    const float w1 = fmaxf(0.f, fmaf(fr - 1.f, t.z, 1.f)) * t.w;
    const T *row = Gs + (size_t)a * ND;
    if (k0 >= 0 && k0 < ND) fma_acc(acc, w0, __ldg(row + k0));
    if (k0 + 1 >= 0 && k0 + 1 < ND) fma_acc(acc, w1, __ldg(row + k0 + 1));
  }
  const size_t q = (size_t)i * N + j;
  const size_t oo = (size_t)s * out_stride + q;
  if constexpr (NMAP == 3) {
    if (mu) {   // cost path: + 2 lambda x (eq. 5); maps have slice stride N*N
      const size_t iq = (size_t)s * N * N + q;
      const float l2 = 2.f * lambda;
      acc.x = fmaf(l2, __ldg(mu + iq), acc.x);
      acc.y = fmaf(l2, __ldg(delta + iq), acc.y);
      acc.z = fmaf(l2, __ldg(sigma + iq), acc.z);
    }
    o0[oo] = acc.x;
    o1[oo] = acc.y;
    o2[oo] = acc.z;
  } else {
    o0[oo] = acc;
  }
}

}  // namespace

template <int NMAP>
static cudaError_t launch_bp(const ei_plan &p, const typename GT<NMAP>::T *G, const float *mu,
                             const float *delta, const float *sigma, float lambda, float *o0,
                             float *o1, float *o2, size_t out_stride, cudaStream_t st) {
  const size_t smem = sizeof(float4) * p.NA;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute((const void *)backproject_kernel<NMAP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((p.N + BX - 1) / BX, (p.N + BY - 1) / BY, p.S), block(BX, BY);
  backproject_kernel<NMAP><<<grid, block, smem, st>>>(G, p.tab.k3, p.N, p.NA, p.ND, mu, delta, sigma,
                                                      lambda, o0, o1, o2, out_stride);
  return cudaGetLastError();
}

cudaError_t launch_backproject3(const ei_plan &p, const float4 *G, const float *mu,
                                const float *delta, const float *sigma, float lambda, float *g_mu,
                                float *g_delta, float *g_sigma, size_t out_stride, cudaStream_t st) {
  return launch_bp<3>(p, G, mu, delta, sigma, lambda, g_mu, g_delta, g_sigma, out_stride, st);
}

cudaError_t launch_backproject1(const ei_plan &p, const float *sino, float *map, cudaStream_t st) {
  return launch_bp<1>(p, sino, nullptr, nullptr, nullptr, 0.f, map, nullptr, nullptr,
                      (size_t)p.N * p.N, st);
}

}  // namespace ei
