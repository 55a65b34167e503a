// k_project.cu — K1: Joseph ray-driven projection (eq. 1; SURVEY.md §8(a) a1,
// readings R5-R8).  Every angle is handled in its dominant-axis frame: row-dominant angles
// sample the rows of the map, column-dominant angles sample the rows of the transposed map
// with (cos, sin) swapped (H2), so the inner loop always walks contiguous rows and the 32
// lanes of a warp (32 adjacent rays of one angle) read adjacent pixels of the same row.
//
// One thread = one ray (s, a, k); it visits only the rows where the ray has a tap inside
// the grid, i.e. |x*_c| < (N+1)/2 with x*_c = (k-(Nd-1)/2)*ic - tn*(i-(N-1)/2).
#include "ei_common.cuh"

namespace ei {
namespace {

template <int NMAP>
struct Pix;
template <>
struct Pix<3> {
  using T = float4;
};
template <>
struct Pix<1> {
  using T = float;
};

__device__ __forceinline__ void row_range(float alpha, float tn, float ctr, int N, int &lo, int &hi) {
  // rows i with |alpha - tn*(i-ctr)| < ctr + 1 (taps inside the grid), conservatively widened
  const float lim = ctr + 1.0f;
  if (fabsf(tn) < 1e-20f) {
    if (fabsf(alpha) < lim + 1.0f) { lo = 0; hi = N - 1; } else { lo = 0; hi = -1; }
    return;
  }
  float y0 = (alpha - lim) / tn, y1 = (alpha + lim) / tn;
  if (y0 > y1) { float t = y0; y0 = y1; y1 = t; }
  const float f0 = floorf(y0 + ctr) - 1.0f, f1 = ceilf(y1 + ctr) + 1.0f;
  lo = f0 < 0.f ? 0 : (f0 > (float)N ? N : (int)f0);
  hi = f1 > (float)(N - 1) ? N - 1 : (f1 < -1.f ? -1 : (int)f1);
}

__device__ __forceinline__ void acc_add(float4 &acc, float4 v0, float4 v1, float w) {
  acc.x += fmaf(w, v1.x - v0.x, v0.x);
  acc.y += fmaf(w, v1.y - v0.y, v0.y);
  acc.z += fmaf(w, v1.z - v0.z, v0.z);
}
__device__ __forceinline__ void acc_add(float &acc, float v0, float v1, float w) {
  acc += fmaf(w, v1 - v0, v0);
}
__device__ __forceinline__ float4 zero_of(float4) { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float zero_of(float) { return 0.f; }

template <int NMAP>
__global__ void __launch_bounds__(128) project_kernel(const typename Pix<NMAP>::T *__restrict__ map,
                                                      const typename Pix<NMAP>::T *__restrict__ mapT,
                                                      const float4 *__restrict__ k1, int N, int NA,
                                                      int ND, float *__restrict__ P) {
  using T = typename Pix<NMAP>::T;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int a = blockIdx.y, s = blockIdx.z;
  if (k >= ND) return;
  const float4 tab = __ldg(k1 + a);   // ic, tn, scale, rowdom
  const size_t NN = (size_t)N * N;
  const T *img = (tab.w != 0.f ? map : mapT) + s * NN;
  const float ctr = 0.5f * (float)(N - 1);
  const float alpha = ((float)k - 0.5f * (float)(ND - 1)) * tab.x;
  int lo, hi;
  row_range(alpha, tab.y, ctr, N, lo, hi);
  T acc = zero_of(T());
  const T zero = zero_of(T());
  for (int i = lo; i <= hi; ++i) {
    const float xs = fmaf(-tab.y, (float)i - ctr, alpha) + ctr;
    const float f = floorf(xs);
    const int j0 = (int)f;
    const float w = xs - f;
    const T *row = img + (size_t)i * N;
    const T v0 = (j0 >= 0 && j0 < N) ? __ldg(row + j0) : zero;
    const T v1 = (j0 + 1 >= 0 && j0 + 1 < N) ? __ldg(row + j0 + 1) : zero;
    acc_add(acc, v0, v1, w);
  }
  const size_t plane = (size_t)NA * ND;
  float *out = P + (size_t)s * NMAP * plane + (size_t)a * ND + k;
  if constexpr (NMAP == 3) {
    out[0] = acc.x * tab.z;
    out[plane] = acc.y * tab.z;
    out[2 * plane] = acc.z * tab.z;
  } else {
    out[0] = acc * tab.z;
  }
}

}  // namespace

cudaError_t launch_project3(const ei_plan &p, float *P, cudaStream_t st) {
  dim3 grid((p.ND + 127) / 128, p.NA, p.S);
  project_kernel<3><<<grid, 128, 0, st>>>(p.maps4, p.maps4T, p.tab.k1, p.N, p.NA, p.ND, P);
  return cudaGetLastError();
}

cudaError_t launch_project1(const ei_plan &p, const float *map, float *P, cudaStream_t st) {
  dim3 grid((p.ND + 127) / 128, p.NA, p.S);
  project_kernel<1><<<grid, 128, 0, st>>>(map, p.mapT1, p.tab.k1, p.N, p.NA, p.ND, P);
  return cudaGetLastError();
}

}  // namespace ei
