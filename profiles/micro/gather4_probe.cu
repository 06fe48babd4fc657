// tile::gather4 probe: four 400-B rows of a 2-D f32 tensor map (d = 100) per
// instruction into shared memory, checked against the table.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__global__ void probe(const __grid_constant__ CUtensorMap tm, const int* rows, float* out, int d,
                      int ngroups, int gstride_floats) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                 "r"(ngroups * 4 * d * 4));
    for (int g = 0; g < ngroups; ++g) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + g * gstride_floats);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
          "l"(&tm), "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]),
          "r"(rows[4 * g + 3]), "r"(b)
          : "memory");
    }
  }
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(b) : "memory");
  for (int g = 0; g < ngroups; ++g)
    for (int i = threadIdx.x; i < 4 * d; i += blockDim.x) out[g * 4 * d + i] = sm[g * gstride_floats + i];
}

int main() {
  const int d = 100, V = 1000003, ngroups = 5;
  const int gstride = getenv("GSTRIDE") ? atoi(getenv("GSTRIDE")) : 416;  // floats per group (416: 1664 B)
  std::vector<float> h((size_t)V * d);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)(i % 1000003) * 0.5f;
  float* dt; cudaMalloc(&dt, h.size() * 4); cudaMemcpy(dt, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  int hr[20] = {5, 17, 3, V - 1, 0, 1, 2, 3, 999, 12345, 777777, 42, 7, 7, 7, 7, 100, 200, 300, 400};
  int* dr; cudaMalloc(&dr, sizeof hr); cudaMemcpy(dr, hr, sizeof hr, cudaMemcpyHostToDevice);
  float* dout; cudaMalloc(&dout, ngroups * 4 * d * 4);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fn;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)V}, strides[1] = {(cuuint64_t)d * 4};
  cuuint32_t box[2] = {(cuuint32_t)d, 1}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dt, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(tm, dr, dout, d, ngroups, gstride);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  std::vector<float> o(ngroups * 4 * d);
  cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int s = 0; s < 20; ++s)
    for (int i = 0; i < d; ++i) bad += o[s * d + i] != h[(size_t)hr[s] * d + i];
  printf("mismatches %d\n", bad);
  return bad != 0 || e != cudaSuccess || r != CUDA_SUCCESS;
}
