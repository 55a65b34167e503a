// tools/smem_wavefronts.cu — shared-memory wavefronts per LDS for the lane->address patterns
// the K1/K3 gathers produce (element sizes 4, 8, 16 B; broadcast and near-contiguous
// patterns).  Run under ncu with
//   --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum
// (one launch per (pattern, size)); also prints cycles per LDS per SM from clock64.
// Design tool, not part of libei.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int pat(int p, int lane) {
  switch (p) {
    case 0: return lane;
    case 1: return lane >> 1;
    case 2: return lane >> 2;
    case 3: return lane >> 3;
    case 4: return lane & 7;
    case 5: return lane & 15;
    case 6: return (lane & 7) + (lane >> 3);           // K3-like 8x4 sub-tile, ~11 entries
    case 7: return (lane & 7) + 2 * (lane >> 3);       // 14 entries
    case 8: return (lane >> 2) + (lane & 3);           // K1-like, 11 entries
    case 9: return 0;
    case 10: return (lane & 3) * 8 + (lane >> 2);      // 32 distinct, quarter = stride 8
    case 11: return lane >> 4;                         // 2 distinct
    default: return lane;
  }
}

template <typename T>
__global__ void lds_kernel(int p, int iters, float *out, long long *cyc) {
  __shared__ __align__(16) T buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    float *f = reinterpret_cast<float *>(&buf[i]);
    for (int q = 0; q < (int)(sizeof(T) / 4); ++q) f[q] = (float)(i + q);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int e = pat(p, lane) + 64 * (threadIdx.x >> 5);
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const T v = buf[(e + u * 32) & 1023];
      const float *f = reinterpret_cast<const float *>(&v);
#pragma unroll
      for (int q = 0; q < (int)(sizeof(T) / 4); ++q) acc += f[q];
    }
    e ^= 1 << 8;   // keep the loads inside the loop (address changes, pattern does not)
  }
  long long t1 = clock64();
  if (acc == 1234.5f) out[0] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  float *out;
  long long *cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, 8);
  const int iters = 2000, blocks = 148 * 4, threads = 512;
  for (int size : {4, 8, 16}) {
    for (int p = 0; p <= 11; ++p) {
      if (size == 4) lds_kernel<float><<<blocks, threads>>>(p, iters, out, cyc);
      if (size == 8) lds_kernel<float2><<<blocks, threads>>>(p, iters, out, cyc);
      if (size == 16) lds_kernel<float4><<<blocks, threads>>>(p, iters, out, cyc);
      long long c = 0;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // cycles per warp-LDS per SM: block 0's elapsed cycles / (LDS per warp x warps per SM)
      const double warps_per_sm = 4.0 * threads / 32;
      printf("size %2d pattern %2d  cyc/LDS/SM %.3f\n", size, p, (double)c / (iters * 8.0 * warps_per_sm));
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
