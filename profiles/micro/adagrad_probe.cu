// Exhaustive-ish check of adagrad_try_fast (csrc/adagrad.cuh) against the
// exact reference update on random operands: every fast-path result must be
// bit-identical; reports the fast-path rate.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2505_09258_b200/csrc/adagrad.cuh"

__device__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull; x ^= x >> 27; x *= 0x94d049bb133111ebull; return x ^ (x >> 31);
}
__device__ double u01(uint64_t& s) { s = mix64(s + 0x9e3779b97f4a7c15ull); return (s >> 11) * 0x1p-53; }

__global__ void probe(uint64_t n, unsigned long long* out, int mode) {
  unsigned long long fast = 0, bad = 0, total = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = i * 0x2545F4914F6CDD1Dull + 7;
    const double r1 = u01(s), r2 = u01(s), r3 = u01(s), r4 = u01(s), r5 = u01(s);
    // theta: mostly the init range, sometimes larger / tiny
    float th = (float)((r1 - 0.5) * (r5 < 0.9 ? 0.1 : (r5 < 0.99 ? 10.0 : 1e-30)));
    // S: zero (first step), small, or accumulated
    float st = r2 < 0.3 ? 0.f : (float)(r3 * (r4 < 0.5 ? 1e-6 : 10.0));
    // gradient: wide magnitude range, both signs, some exact zeros / cancellations
    double g = (r4 - 0.5) * exp2(-60.0 * r3 + 2.0);
    if (r5 > 0.999) g = 0.0;
    const double lr = 0.1, eps = 1e-10;
    float th_e = th, st_e = st, th_f = th, st_f = st;
    lgd::adagrad_exact(g, th_e, st_e, lr, eps);
    const bool ok = mode ? lgd::adagrad_try_fast1(g, th_f, st_f, lr, eps)
                         : lgd::adagrad_try_fast(g, th_f, st_f, lr, eps);
    ++total;
    if (ok) {
      ++fast;
      if (__float_as_uint(th_f) != __float_as_uint(th_e) || __float_as_uint(st_f) != __float_as_uint(st_e)) ++bad;
    }
  }
  atomicAdd(out, total); atomicAdd(out + 1, fast); atomicAdd(out + 2, bad);
}

int main(int argc, char** argv) {
  const unsigned long long n = argc > 1 ? strtoull(argv[1], nullptr, 0) : (1ull << 32);
  unsigned long long* d; cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
  const int mode = argc > 2 ? atoi(argv[2]) : 0;  // 1: the single-Newton-step variant
  probe<<<148 * 8, 256>>>(n, d, mode);
  unsigned long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("%s total %llu fast %llu (%.5f%%) mismatches %llu\n", cudaGetErrorString(cudaGetLastError()),
         h[0], h[1], 100.0 * h[1] / h[0], h[2]);
  return h[2] != 0;
}
