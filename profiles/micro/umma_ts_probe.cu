// Probe: tcgen05.mma kind::tf32 with A in TMEM ("TS"), A placed there either
// by tcgen05.cp from the no-swizzle K-major core-matrix layout in shared
// memory (mode 0) or by tcgen05.st from registers, thread = row (mode 1).
// D[128 x N] = A[128 x K] . B[N x K]^T, B K-major in shared memory.
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
__host__ __device__ constexpr uint32_t instr_desc(uint32_t M, uint32_t N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ uint32_t cm(uint32_t r, uint32_t c, uint32_t cols) {
  return ((r >> 3) * (cols >> 2) + (c >> 2)) * 128 + (r & 7) * 16 + (c & 3) * 4;
}

template <int K, int N>
__global__ void probe(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  unsigned char* sA = sm;
  unsigned char* sB = sm + 128 * K * 4;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * K; i += blockDim.x) *(float*)(sA + cm(i / K, i % K, K)) = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) *(float*)(sB + cm(i / K, i % K, K)) = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tb)), "r"(512));
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
  const uint32_t a_tm = t + 256;  // A at columns [256, 256 + K)
  if (mode == 1) {  // thread = row: its K values into lane `tid`, 8 columns at a time
    for (int c = 0; c < K; c += 8) {
      uint32_t v[8];
      for (int e = 0; e < 8; ++e) v[e] = __float_as_uint(A[tid * K + c + e]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::
                   "r"(a_tm + ((uint32_t)(warp * 32) << 16) + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
                   "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t kcore = (K / 4) * 128;
    if (mode == 0) {
      for (int ks = 0; ks < K / 8; ++ks)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(a_tm + ks * 8),
                     "l"(smem_desc(saddr(sA) + ks * 256, 128, kcore)) : "memory");
    }
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t bd = smem_desc(saddr(sB) + ks * 256, 128, kcore);
      uint32_t acc = ks > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t),
                   "r"(a_tm + ks * 8), "l"(bd), "r"(instr_desc(128, N)), "r"(acc));
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}


template <int N>
__global__ void rate(unsigned long long* out, int reps, int ss) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (128 + N) * 8; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(&tb)), "r"(512));
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
    const uint64_t ad = smem_desc(saddr(sm), 128, 256);
    const uint64_t bd = smem_desc(saddr(sm) + 128 * 32, 128, 256);
    const uint32_t id = instr_desc(128, N);
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (ss)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(t), "l"(ad), "l"(bd), "r"(id), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(t), "r"(t + 256), "l"(bd), "r"(id), "r"(1));
    }
    unsigned long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(saddr(&bar)));
    unsigned long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}
template <int N> void run_rate(unsigned long long* d) {
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ss = 0; ss < 2; ++ss) {
    rate<N><<<1, 128, 64 * 1024>>>(d, 1000, ss);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d %s: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", N, ss ? "SS" : "TS", h[0] / 1000.0, h[1] / 1000.0,
           cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  { unsigned long long* dd; cudaMalloc(&dd, 16); run_rate<64>(dd); run_rate<128>(dd); run_rate<256>(dd); }
  constexpr int K = 112, N = 64;
  std::vector<float> A(128 * K), B(N * K), D(128 * N), ref(128 * N);
  srand(1);
  for (auto& x : A) x = (rand() % 17 - 8) / 8.0f;
  for (auto& x : B) x = (rand() % 17 - 8) / 8.0f;
  for (int i = 0; i < 128; ++i)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[i * K + k] * B[n * K + k];
      ref[i * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  size_t smem = 128 * K * 4 + N * K * 4;
  cudaFuncSetAttribute(probe<K, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<K, N><<<1, 128, smem>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (size_t i = 0; i < D.size(); ++i) err = fmax(err, fabs(D[i] - ref[i]));
    printf("mode %d (%s): %s max|err| = %g  D[0..2] = %g %g %g  ref %g %g %g\n", mode,
           mode ? "tcgen05.st" : "tcgen05.cp", cudaGetErrorString(e), err, D[0], D[1], D[2], ref[0], ref[1], ref[2]);
    if (e != cudaSuccess) return 1;
    fails += err > 0;
  }
  return fails;
}
