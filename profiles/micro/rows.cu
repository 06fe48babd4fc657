// Microbenchmark (not product): cost decomposition of the K4 row update.
// 1.56M sorted unique rows out of 7.8M (a TW batch), d = 100, warp per row,
// float4 lanes.  (a) theta/S read + write, (b) + FP64 Adagrad, (c) + one
// snapshot-row gather + contribution math, (d) (c) with 2 rows per warp.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ void adagrad(double g, float& th, float& st) {
  const double acc = (double)st + g * g;
  st = (float)acc;
  const double num = 0.1 * g;
  th = (float)((double)th - num / (sqrt(acc) + 1e-10));
}

template <int MODE>
__global__ void __launch_bounds__(256) rows_kernel(const uint32_t* __restrict__ rows, uint64_t nrows,
                                                   float* __restrict__ th, float* __restrict__ st,
                                                   const float* __restrict__ snap, uint32_t P) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = ((uint64_t)blockIdx.x * 256 + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t)gridDim.x * 8;
  for (uint64_t i = w; i < nrows; i += nw) {
    const uint64_t r = rows[i];
    if (lane >= 25) continue;
    float4 t = *reinterpret_cast<const float4*>(th + r * 100 + 4 * lane);
    float4 s = *reinterpret_cast<const float4*>(st + r * 100 + 4 * lane);
    double g[4] = {1e-3 * (lane + 1), -2e-3, 3e-4, -4e-4};
    if (MODE >= 2) {
      const uint64_t p = (r * 2654435761ull) % P;
      const float4 sv = __ldg(reinterpret_cast<const float4*>(snap + p * 100 + 4 * lane));
      g[0] += 0.3 * (double)sv.x; g[1] += 0.3 * (double)sv.y; g[2] += 0.3 * (double)sv.z; g[3] += 0.3 * (double)sv.w;
    }
    if (MODE >= 1) {
      adagrad(g[0], t.x, s.x); adagrad(g[1], t.y, s.y); adagrad(g[2], t.z, s.z); adagrad(g[3], t.w, s.w);
    } else {
      t.x += 1.f; s.x += 1.f;
    }
    *reinterpret_cast<float4*>(th + r * 100 + 4 * lane) = t;
    *reinterpret_cast<float4*>(st + r * 100 + 4 * lane) = s;
  }
}

int main() {
  const uint64_t V = 7800000, N = 1560000, d = 100; const uint32_t P = 100000;
  std::vector<uint32_t> all(V); for (uint64_t i = 0; i < V; ++i) all[i] = i;
  std::mt19937_64 g(1); std::shuffle(all.begin(), all.end(), g);
  std::vector<uint32_t> rows(all.begin(), all.begin() + N); std::sort(rows.begin(), rows.end());
  float *th, *st, *snap; uint32_t* dr;
  cudaMalloc(&th, V * d * 4); cudaMalloc(&st, V * d * 4); cudaMalloc(&snap, P * d * 4); cudaMalloc(&dr, N * 4);
  cudaMemset(th, 0, V * d * 4); cudaMemset(st, 0, V * d * 4); cudaMemset(snap, 0, P * d * 4);
  cudaMemcpy(dr, rows.data(), N * 4, cudaMemcpyHostToDevice);
  float* flush; cudaMalloc(&flush, 512ull << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 3; ++mode) {
    for (int grid_mult : {4, 8, 16, 64}) {
      const int grid = sms * grid_mult;
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 512ull << 20);
        cudaEventRecord(a);
        if (mode == 0) rows_kernel<0><<<grid, 256>>>(dr, N, th, st, snap, P);
        if (mode == 1) rows_kernel<1><<<grid, 256>>>(dr, N, th, st, snap, P);
        if (mode == 2) rows_kernel<2><<<grid, 256>>>(dr, N, th, st, snap, P);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
      }
      const double bytes = (double)N * 1600;
      printf("mode %d grid %4d x256: %.3f ms  %.0f GB/s (algorithmic 16d/row)\n", mode, grid, best, bytes / best / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
