// tools/microbench.cu — measures the on-chip roofline denominators used in DESIGN.md §6 on
// the B200 box: L2 read bandwidth (L2-resident buffer), shared-memory LDS.128 bandwidth, and
// HBM read bandwidth (buffer >> L2).  Prints one JSON line.  Not part of libei.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_kernel(const float4* __restrict__ p, size_t n, int passes, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < passes; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

__global__ void smem_kernel(int iters, float* out) {
  __shared__ float4 buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4 v = buf[(idx + u * 256) & 2047];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    idx += 32;
  }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}

int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  // L2: 48 MB resident buffer, read many passes
  size_t n2 = 48ull << 20; float4* p2; cudaMalloc(&p2, n2); cudaMemset(p2, 0, n2);
  int grid = prop.multiProcessorCount * 8;
  read_kernel<<<grid, 256>>>(p2, n2 / 16, 2, out);
  cudaEventRecord(a); read_kernel<<<grid, 256>>>(p2, n2 / 16, 40, out); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  double l2 = 40.0 * n2 / (ms * 1e-3) / 1e9;
  // HBM: 4 GB buffer, one pass
  size_t nh = 4ull << 30; float4* ph; cudaMalloc(&ph, nh); cudaMemset(ph, 0, nh);
  read_kernel<<<grid, 256>>>(ph, nh / 16, 1, out);
  cudaEventRecord(a); read_kernel<<<grid, 256>>>(ph, nh / 16, 2, out); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  double hbm = 2.0 * nh / (ms * 1e-3) / 1e9;
  // SMEM: LDS.128, conflict-free, 8 blocks x 256 threads per SM
  int iters = 20000;
  smem_kernel<<<prop.multiProcessorCount * 4, 256>>>(10, out);
  cudaEventRecord(a); smem_kernel<<<prop.multiProcessorCount * 4, 256>>>(iters, out); cudaEventRecord(b);
  cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  double sm_bytes = (double)prop.multiProcessorCount * 4 * 256 * iters * 8 * 16;
  double smem = sm_bytes / (ms * 1e-3) / 1e9;
  printf("{\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"smem_lds128_gbs\": %.1f, \"sms\": %d, \"clock_khz_attr\": %d}\n",
         l2, hbm, smem, prop.multiProcessorCount, clk_khz);
  return 0;
}
