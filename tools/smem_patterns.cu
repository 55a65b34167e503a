// tools/smem_patterns.cu — shared-memory wavefronts per LDS for candidate lane->pixel (K3) and
// lane->(angle, ray) (K1) mappings evaluated on real geometry.  One launch per (mapping, element
// size); ncu's l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum /
// smsp__sass_inst_executed_op_shared_ld.sum gives the average wavefronts per LDS for it.
// Design tool, not part of libei.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int NPAT = 512;

template <typename T>
__global__ void run(const int *__restrict__ pats, int iters, float *out) {
  __shared__ __align__(16) T buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
    float *f = reinterpret_cast<float *>(&buf[i]);
    for (int q = 0; q < (int)(sizeof(T) / 4); ++q) f[q] = (float)(i + q);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int p = (blockIdx.x * 16 + w * 4 + it) % NPAT;
    const int e = pats[p * 32 + lane] + 128 * (it & 7);
    const T v = buf[e];
    const float *f = reinterpret_cast<const float *>(&v);
#pragma unroll
    for (int q = 0; q < (int)(sizeof(T) / 4); ++q) acc += f[q];
  }
  if (acc == 1234.5f) out[0] = acc;
}

// K3 mappings: lane -> (px, py) inside the warp's footprint
static void k3_map(int m, int lane, int &px, int &py) {
  switch (m) {
    case 0: px = lane & 7; py = lane >> 3; break;                    // current 8x4
    case 1: px = lane & 3; py = lane >> 2; break;                    // 4x8
    case 2: px = lane & 15; py = lane >> 4; break;                   // 16x2
    case 3: px = lane; py = 0; break;                                // 32x1
    case 4: px = lane >> 3; py = lane & 7; break;                    // 4x8 column-major
    case 5: px = (lane & 1) | (((lane >> 2) & 1) << 1);               // 4x8 in 2x2 Morton blocks
            py = ((lane >> 1) & 1) | ((lane >> 3) << 1); break;
    case 6: px = (lane & 7) >> 1; py = (lane >> 3) * 2 + (lane & 1); break;   // 4x8 in 2x2 blocks
    default: px = lane & 7; py = lane >> 3;
  }
}

int main(int argc, char **argv) {
  int *d;
  float *out;
  cudaMalloc(&d, NPAT * 32 * sizeof(int));
  cudaMalloc(&out, 4);
  std::vector<int> h(NPAT * 32);
  srand(1);
  // ---- K3: pixel gather of detector entries, du = dx = 1 ----
  for (int m = 0; m <= 6; ++m) {
    for (int p = 0; p < NPAT; ++p) {
      const double th = M_PI * (p + 0.37) / NPAT;
      const double c = cos(th), s = sin(th);
      const double ox = (rand() % 1000) / 7.3, oy = (rand() % 1000) / 9.1;
      int mn = 1 << 30;
      int k[32];
      for (int l = 0; l < 32; ++l) {
        int px, py;
        k3_map(m, l, px, py);
        k[l] = (int)floor((ox + px) * c + (oy + py) * s + 1000.0);
        mn = k[l] < mn ? k[l] : mn;
      }
      for (int l = 0; l < 32; ++l) h[p * 32 + l] = k[l] - mn;
    }
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    run<float><<<148 * 2, 512>>>(d, 4000, out);
    run<float2><<<148 * 2, 512>>>(d, 4000, out);
    run<float4><<<148 * 2, 512>>>(d, 4000, out);
    printf("k3 mapping %d launched (float, float2, float4)\n", m);
  }
  // ---- rule probes for 8-byte loads ----
  for (int m = 0; m < 6; ++m) {
    for (int p = 0; p < NPAT; ++p)
      for (int l = 0; l < 32; ++l) {
        int e = 0;
        switch (m) {
          case 0: e = (l & 15) >> 1; break;              // halves identical, adjacent duplicates
          case 1: e = l & 1; break;                      // 2 entries everywhere
          case 2: e = (l & 7) + 8 * (l >> 4); break;     // halves disjoint, duplicates at +8
          case 3: e = (l >> 1) + (l >> 4); break;        // lane>>1, half 1 shifted by one entry
          case 4: e = (l & 15) >> 2; break;              // halves identical, 4 entries
          case 5: e = (l >> 2) + 2 * (l >> 4); break;    // 8 entries + half 1 shifted by 2
        }
        h[p * 32 + l] = e;
      }
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    run<float2><<<148 * 2, 512>>>(d, 4000, out);
    run<float4><<<148 * 2, 512>>>(d, 4000, out);
    printf("probe %d launched (float2, float4)\n", m);
  }
  if (argc > 2) {   // K1 patterns for a given angle step (deg) and N: angle-fast and ray-fast
    const double stepdeg = atof(argv[1]);
    const int Nmap = atoi(argv[2]);
    for (int m = 0; m < 2; ++m) {
      for (int p = 0; p < NPAT; ++p) {
        const double th0 = (M_PI / 2) * (p + 0.5) / NPAT - M_PI / 4;
        const double step = stepdeg * M_PI / 180;
        const double y = (rand() % Nmap) - Nmap / 2.0;
        const double r0 = (rand() % Nmap) - Nmap / 2.0;
        int mn = 1 << 30;
        int k[32];
        for (int l = 0; l < 32; ++l) {
          const int a = m == 0 ? (l & 3) : (l >> 3), r = m == 0 ? (l >> 2) : (l & 7);
          const double th = th0 + a * step, c = cos(th), s = sin(th);
          k[l] = (int)floor((r0 + r) / c - y * s / c + 4000.0);
          mn = k[l] < mn ? k[l] : mn;
        }
        for (int l = 0; l < 32; ++l) h[p * 32 + l] = k[l] - mn;
      }
      cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
      run<float2><<<148 * 2, 512>>>(d, 4000, out);
      run<float4><<<148 * 2, 512>>>(d, 4000, out);
      printf("sweep step %g N %d mapping %d launched (float2, float4)\n", stepdeg, Nmap, m);
    }
    cudaDeviceSynchronize();
    return 0;
  }
  // ---- K1: lane -> (angle a of 16 adjacent angles at 0.25 deg, ray r), row y ----
  // x*(a, r, y) = r / cos - y tan + ctr, pair entry floor(x*)
  for (int m = 0; m <= 4; ++m) {
    for (int p = 0; p < NPAT; ++p) {
      const double th0 = (M_PI / 4) * (p + 0.5) / NPAT - M_PI / 8;   // row-dominant range
      const double step = M_PI / 720;
      const double y = (rand() % 512) - 256.0;
      const double r0 = (rand() % 512) - 256.0;
      int mn = 1 << 30;
      int k[32];
      for (int l = 0; l < 32; ++l) {
        int a, r;
        switch (m) {
          case 0: a = l & 3; r = l >> 2; break;        // current: 4 angles x 8 rays (angle fastest)
          case 1: a = 0; r = l; break;                 // 1 angle x 32 rays
          case 2: a = l >> 3; r = l & 7; break;        // 4 angles x 8 rays (ray fastest)
          case 3: a = l & 7; r = l >> 3; break;        // 8 angles x 4 rays
          case 4: a = l >> 4; r = l & 15; break;       // 2 angles x 16 rays
          default: a = 0; r = l;
        }
        const double th = th0 + a * step, c = cos(th), s = sin(th);
        k[l] = (int)floor((r0 + r) / c - y * s / c + 2000.0);
        mn = k[l] < mn ? k[l] : mn;
      }
      for (int l = 0; l < 32; ++l) h[p * 32 + l] = k[l] - mn;
    }
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    run<float><<<148 * 2, 512>>>(d, 4000, out);
    run<float2><<<148 * 2, 512>>>(d, 4000, out);
    run<float4><<<148 * 2, 512>>>(d, 4000, out);
    printf("k1 mapping %d launched (float, float2, float4)\n", m);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
