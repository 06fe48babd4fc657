// Probe: tcgen05.mma kind::tf32 with a K-major A and an MN-major B held in the
// no-swizzle core-matrix layout, for both LBO/SBO assignments.  D = A B,
// A [128 x K] (K-major), B given as [K x N] rows with N contiguous.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t instr_desc(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ uint32_t cm(uint32_t r, uint32_t c, uint32_t cols) {
  return ((r >> 3) * (cols >> 2) + (c >> 2)) * 128 + (r & 7) * 16 + (c & 3) * 4;
}

// mode 0: B K-major (B^T stored [N x K] in core layout)
// mode 1: B MN-major from [K x N] core layout, lbo = K-group stride, sbo = 128
// mode 2: B MN-major, lbo = 128, sbo = K-group stride
__global__ void probe(const float* A, const float* B, float* D, int K, int N, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  unsigned char* sA = sm;
  unsigned char* sB = sm + 128 * K * 4;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * K; i += blockDim.x) {
    int r = i / K, c = i % K;
    *(float*)(sA + cm(r, c, K)) = A[i];
  }
  for (int i = tid; i < K * N; i += blockDim.x) {
    int kk = i / N, n = i % N;  // B[k][n]
    if (mode == 0) *(float*)(sB + cm(n, kk, K)) = B[i];   // [N x K] rows of K
    else *(float*)(sB + cm(kk, n, N)) = B[i];             // [K x N] rows of N
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tb)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = tb;
  if (tid == 0) {
    const uint32_t kcoreA = (K / 4) * 128;
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t ad = smem_desc(saddr(sA) + ks * 256, 128, kcoreA);
      uint64_t bd;
      if (mode == 0) bd = smem_desc(saddr(sB) + ks * 256, 128, kcoreA);
      else {
        const uint32_t kg = (N / 4) * 128;  // next 8 K-rows
        bd = mode == 1 ? smem_desc(saddr(sB) + ks * kg, kg, 128) : smem_desc(saddr(sB) + ks * kg, 128, kg);
      }
      uint32_t id = instr_desc(128, N, false, mode != 0);
      uint32_t acc = ks > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(t), "l"(ad), "l"(bd), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
  }
  uint32_t ok = 0;
  while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(saddr(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(t + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int e = 0; e < 16; ++e) D[tid * N + c + e] = __uint_as_float(r[e]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(256));
}

int main() {
  const int K = 64, N = 112;
  std::vector<float> A(128 * K), B(K * N), D(128 * N), ref(128 * N);
  srand(1);
  for (auto& x : A) x = (rand() % 17 - 8) / 8.0f;
  for (auto& x : B) x = (rand() % 17 - 8) / 8.0f;
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[k * N + n];
      ref[i * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  size_t smem = 128 * K * 4 + K * N * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, K, N, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (size_t i = 0; i < D.size(); ++i) err = fmax(err, fabs(D[i] - ref[i]));
    printf("mode %d: %s max|err| = %g  D[0..3] = %g %g %g  ref %g %g %g\n", mode, cudaGetErrorString(e), err,
           D[0], D[1], D[2], ref[0], ref[1], ref[2]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
