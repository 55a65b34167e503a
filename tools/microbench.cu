// tools/microbench.cu — measures the on-chip roofline denominators used by bench.py for K1/K3
// on the B200 box: shared-memory LDS.128 and LDS.64 bandwidth (conflict-free,
// every lane a distinct address), L2 read bandwidth (L2-resident 48 MB buffer) and HBM read
// bandwidth (4 GiB buffer >> L2).  Each figure is the best of 5 timed launches of ~0.1-1 s
// (CUDA events).  Prints one JSON line; tools/measure_peaks.py runs it under an nvidia-smi
// clock sampler and writes profiles/r02/peaks.json.  Not part of libei.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_kernel(const float4* __restrict__ p, size_t n, int passes, float* out,
                            long long* cyc) {
  const long long c0 = clock64();
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < passes; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

// T = float4 (LDS.128) or float2 (LDS.64): lane l of a warp reads element (base + l) — a quarter
// (LDS.128) or half (LDS.64) warp covers 128 contiguous bytes, one wavefront each
template <typename T>
__global__ void smem_kernel(int iters, float* out, long long* cyc) {
  __shared__ T buf[2048];
  const long long c0 = clock64();
  float* f = reinterpret_cast<float*>(buf);
  for (int i = threadIdx.x; i < 2048 * (int)(sizeof(T) / 4); i += blockDim.x) f[i] = (float)i;
  __syncthreads();
  T acc;
  float* a = reinterpret_cast<float*>(&acc);
  for (int q = 0; q < (int)(sizeof(T) / 4); ++q) a[q] = 0.f;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      T v = buf[(idx + u * 256) & 2047];
      const float* b = reinterpret_cast<const float*>(&v);
#pragma unroll
      for (int q = 0; q < (int)(sizeof(T) / 4); ++q) a[q] += b[q];
    }
    idx += 32;
  }
  float s = 0.f;
  for (int q = 0; q < (int)(sizeof(T) / 4); ++q) s += a[q];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - c0;
}

// mean SM cycles of a launch's blocks (each block's own clock64 span; blocks of one launch run
// concurrently, so this is the kernel's duration in SM clocks)
static double mean_cycles(const long long* d, int n) {
  static long long h[1 << 16];
  cudaMemcpy(h, d, sizeof(long long) * n, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < n; ++i) s += (double)h[i];
  return s / n;
}

// SM clock under load: every block spins for a fixed number of its SM's clock64 cycles; the event
// time of the launch gives the clock rate (the spin keeps the SMs busy, so DVFS sees load)
__global__ void clock_kernel(long long cycles, float* out) {
  const long long t0 = clock64();
  long long t = t0;
  while (t - t0 < cycles) t = clock64();
  if (t == 42) out[0] = 1.f;
}

template <typename F>
static double best_ms(F launch, int reps = 5) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();   // warm-up
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    float ms;
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  const int sms = prop.multiProcessorCount;
  float* out;
  cudaMalloc(&out, 4);
  long long* cyc;
  cudaMalloc(&cyc, sizeof(long long) * (1 << 16));
  // L2: 48 MB resident buffer (fits either die's half of the 126 MB L2), 40 passes per launch
  const size_t n2 = 48ull << 20;
  float4* p2;
  cudaMalloc(&p2, n2);
  cudaMemset(p2, 0, n2);
  const int grid = sms * 8;
  double ms = best_ms([&] { read_kernel<<<grid, 256>>>(p2, n2 / 16, 40, out, cyc); });
  const double l2 = 40.0 * n2 / (ms * 1e-3) / 1e9;
  const double l2_mhz = mean_cycles(cyc, grid) / (ms * 1e3);   // last launch (~ the best one)
  // HBM: 4 GiB buffer, 8 passes per launch
  const size_t nh = 4ull << 30;
  float4* ph;
  cudaMalloc(&ph, nh);
  cudaMemset(ph, 0, nh);
  ms = best_ms([&] { read_kernel<<<grid, 256>>>(ph, nh / 16, 8, out, cyc); });
  const double hbm = 8.0 * nh / (ms * 1e-3) / 1e9;
  // SMEM: 4 CTAs x 256 threads per SM, 8 loads per iteration
  const int iters = 20000;
  const double nload = (double)sms * 4 * 256 * iters * 8;
  ms = best_ms([&] { smem_kernel<float4><<<sms * 4, 256>>>(iters, out, cyc); });
  const double lds128 = nload * 16 / (ms * 1e-3) / 1e9;
  const double c128 = mean_cycles(cyc, sms * 4);
  const double lds128_bpc = nload * 16 / sms / c128;            // bytes per SM clock
  const double smem_mhz = c128 / (ms * 1e3);
  ms = best_ms([&] { smem_kernel<float2><<<sms * 4, 256>>>(iters, out, cyc); });
  const double lds64 = nload * 8 / (ms * 1e-3) / 1e9;
  const double lds64_bpc = nload * 8 / sms / mean_cycles(cyc, sms * 4);
  // SM clock under load (right after the shared-memory runs): cycles / time of a spin launch
  const long long spin = 400000000LL;
  ms = best_ms([&] { clock_kernel<<<sms * 4, 32>>>(spin, out); }, 3);
  const double spin_mhz = (double)spin / (ms * 1e3);
  const cudaError_t e = cudaDeviceSynchronize();
  printf("{\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"smem_lds128_gbs\": %.1f, "
         "\"smem_lds64_gbs\": %.1f, \"blockspan_lds128_bytes_per_sm_clk\": %.2f, "
         "\"blockspan_lds64_bytes_per_sm_clk\": %.2f, \"blockspan_mhz_smem\": %.1f, "
         "\"blockspan_mhz_l2\": %.1f, \"sm_mhz_spin\": %.1f, \"sms\": %d, \"cuda\": \"%s\"}\n",
         l2, hbm, lds128, lds64, lds128_bpc, lds64_bpc, smem_mhz, l2_mhz, spin_mhz, sms, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
