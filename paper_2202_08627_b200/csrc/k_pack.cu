// k_pack.cu — K0: pack the three maps into float4 (mu, delta, sigma, 0) in row-major and
// transposed order (hard part H2: column-dominant angles read the
// transposed copy so every projector load runs along a contiguous row), count non-finite
// inputs into status[0], and emit per-tile sum(x^2) partials for the eq. 5 regulariser.
#include "ei_common.cuh"

namespace ei {
namespace {

constexpr int TILE = 32;

// grid (ceil(N/32), ceil(N/32), S), block (32, 8)
__global__ void __launch_bounds__(256) pack3_kernel(const float *__restrict__ mu,
                                                    const float *__restrict__ delta,
                                                    const float *__restrict__ sigma,
                                                    size_t in_stride, int N,
                                                    float4 *__restrict__ out,
                                                    float4 *__restrict__ outT,
                                                    double *__restrict__ part_reg,
                                                    int32_t *__restrict__ status) {
  __shared__ float4 tile[TILE][TILE + 1];
  __shared__ double red[8];
  const int s = blockIdx.z;
  const int i0 = blockIdx.y * TILE, j0 = blockIdx.x * TILE;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const size_t NN = (size_t)N * N;
  const float *m = mu + s * in_stride, *d = delta + s * in_stride, *g = sigma + s * in_stride;
  float4 *o = out + s * NN, *oT = outT + s * NN;
  double sq = 0.0;
  int bad = 0;
  for (int r = ty; r < TILE; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    if (i < N && j < N) {
      const size_t q = (size_t)i * N + j;
      const float a = __ldg(m + q), b = __ldg(d + q), c = __ldg(g + q);
      bad += !isfinite(a) + !isfinite(b) + !isfinite(c);
      sq += (double)a * a + (double)b * b + (double)c * c;
      const float4 v = make_float4(a, b, c, 0.f);
      o[q] = v;
      tile[r][tx] = v;
    }
  }
  __syncthreads();
  for (int r = ty; r < TILE; r += 8) {
    const int jj = j0 + r, ii = i0 + tx;   // write row jj of the transpose
    if (jj < N && ii < N) oT[(size_t)jj * N + ii] = tile[tx][r];
  }
  if (status && bad) atomicAdd(&status[0], bad);   // integer count: order-independent
  if (part_reg) {
    for (int off = 16; off > 0; off >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, off);
    if (tx == 0) red[ty] = sq;
    __syncthreads();
    if (ty == 0 && tx == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      part_reg[(size_t)s * gridDim.x * gridDim.y + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
  }
}

// single map [S][N][N] (slice stride NN) -> transposed copy
__global__ void __launch_bounds__(256) transpose1_kernel(const float *__restrict__ in, int N,
                                                         float *__restrict__ outT) {
  __shared__ float tile[TILE][TILE + 1];
  const int s = blockIdx.z;
  const int i0 = blockIdx.y * TILE, j0 = blockIdx.x * TILE;
  const size_t NN = (size_t)N * N;
  for (int r = threadIdx.y; r < TILE; r += 8) {
    const int i = i0 + r, j = j0 + threadIdx.x;
    if (i < N && j < N) tile[r][threadIdx.x] = __ldg(in + s * NN + (size_t)i * N + j);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < TILE; r += 8) {
    const int jj = j0 + r, ii = i0 + threadIdx.x;
    if (jj < N && ii < N) outT[s * NN + (size_t)jj * N + ii] = tile[threadIdx.x][r];
  }
}

// sino [S][3][NA*ND] -> float4 [S][NA*ND]
__global__ void pack_sino3_kernel(const float *__restrict__ in, size_t plane, int S,
                                  float4 *__restrict__ out) {
  const size_t total = plane * S;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < total;
       t += (size_t)gridDim.x * blockDim.x) {
    const size_t s = t / plane, q = t - s * plane;
    const float *b = in + s * 3 * plane + q;
    out[t] = make_float4(__ldg(b), __ldg(b + plane), __ldg(b + 2 * plane), 0.f);
  }
}

__global__ void check_small_kernel(const float *__restrict__ flat, int nflat,
                                   const float *__restrict__ mask, int M,
                                   const float *__restrict__ drift, int NA,
                                   int32_t *__restrict__ status) {
  int bad = 0;
  const int total = nflat + M + (drift ? NA : 0);
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    float v = t < nflat ? flat[t] : (t < nflat + M ? mask[t - nflat] : drift[t - nflat - M]);
    bad += !isfinite(v);
  }
  for (int off = 16; off > 0; off >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, off);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(&status[0], bad);
}

}  // namespace

cudaError_t launch_pack3(const ei_plan &p, const float *mu, const float *delta, const float *sigma,
                         size_t in_stride, bool want_reg, int32_t *status, cudaStream_t st) {
  dim3 grid((p.N + TILE - 1) / TILE, (p.N + TILE - 1) / TILE, p.S), block(32, 8);
  pack3_kernel<<<grid, block, 0, st>>>(mu, delta, sigma, in_stride, p.N, p.maps4, p.maps4T,
                                       want_reg ? p.part_reg : nullptr, status);
  return cudaGetLastError();
}

cudaError_t launch_transpose1(const ei_plan &p, const float *map, cudaStream_t st) {
  dim3 grid((p.N + TILE - 1) / TILE, (p.N + TILE - 1) / TILE, p.S), block(32, 8);
  transpose1_kernel<<<grid, block, 0, st>>>(map, p.N, p.mapT1);
  return cudaGetLastError();
}

cudaError_t launch_pack_sino3(const ei_plan &p, const float *sino, cudaStream_t st) {
  const size_t plane = (size_t)p.NA * p.ND;
  const size_t total = plane * p.S;
  const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16);
  pack_sino3_kernel<<<blocks, 256, 0, st>>>(sino, plane, p.S, p.sino4);
  return cudaGetLastError();
}

cudaError_t launch_check_small(const ei_plan &p, const float *flat, const float *mask,
                               const float *drift, int32_t *status, cudaStream_t st) {
  const int nflat = p.S * 3 * p.ND;
  const int total = nflat + p.M + p.NA;
  const int blocks = (total + 255) / 256 < 64 ? (total + 255) / 256 : 64;
  check_small_kernel<<<blocks, 256, 0, st>>>(flat, nflat, mask, p.M, drift, p.NA, status);
  return cudaGetLastError();
}

}  // namespace ei
