// shuffle.cu -- K1: the per-bucket Fisher-Yates shuffle of pipeline.cpp:297-301
// ("for i = m..2: swap(e[i-1], e[next_below(i)])") as a data-parallel
// permutation construction, exact for any draw sequence.
//
// With 0-based steps t = m-1..1 swapping A[t] and A[H[t]] (H[t] <= t), let
// T_q = {t > q : H[t] = q} be the steps that reach position q from above.
//  * G(q), the value at q just before step q runs (q is final afterwards),
//    is G(min T_q) if T_q is non-empty, else the original element q.
//  * Step t writes G(t) into H[t], and the final element at t is whatever
//    H[t] held before step t: G(t') for the next-larger t' in T_{H[t]},
//    else the original element H[t]; a self swap (H[t] = t) leaves G(t);
//    position 0 ends with G(0).
// A stable radix sort of (H[t], t) gives every T_q in ascending order; G is
// resolved by following the strictly increasing chains q -> min T_q.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "internal.hpp"

namespace lgd {

namespace {

constexpr int kThreads = 256;

__global__ void keys_kernel(const uint32_t* __restrict__ H, uint64_t m,
                            uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;  // 1..m-1
  if (t >= m) return;
  const uint32_t h = H[t];
  keys[t - 1] = h < t ? h : (uint32_t)m;  // self swaps sort last (sentinel m)
  vals[t - 1] = (uint32_t)t;
}

__global__ void head_kernel(const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
                            uint64_t n, uint32_t sentinel, uint32_t* __restrict__ ptr) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t q = skeys[s];
  if (q == sentinel) return;
  if (s == 0 || skeys[s - 1] != q) ptr[q] = svals[s];  // min T_q
}

__global__ void chase_kernel(const uint32_t* __restrict__ ptr, uint64_t m, uint32_t* __restrict__ G) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  uint32_t x = (uint32_t)p;
  for (uint32_t nx = ptr[x]; nx != kNone32; nx = ptr[x]) x = nx;
  G[p] = x;
}

__global__ void final_kernel(const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
                             uint64_t n, uint32_t sentinel, const uint32_t* __restrict__ G,
                             uint32_t* __restrict__ perm) {
  const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t q = skeys[s];
  const uint32_t t = svals[s];
  if (q == sentinel) {
    perm[t] = G[t];  // self swap
    return;
  }
  perm[t] = (s + 1 < n && skeys[s + 1] == q) ? G[svals[s + 1]] : q;
}

__global__ void zero_kernel(const uint32_t* __restrict__ G, uint32_t* __restrict__ perm) {
  perm[0] = G[0];
}

__global__ void gather_edges_kernel(const uint32_t* __restrict__ edges,
                                    const uint32_t* __restrict__ perm, uint64_t m,
                                    uint32_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t src = perm ? perm[i] : i;
  out[3 * i] = edges[3 * src];
  out[3 * i + 1] = edges[3 * src + 1];
  out[3 * i + 2] = edges[3 * src + 2];
}

}  // namespace

size_t shuffle_sort_temp_bytes(uint64_t m_max) {
  size_t bytes = 0;
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (int64_t)(m_max ? m_max : 1), 0,
                                           32));
  return bytes;
}

void launch_shuffle_permutation(const uint32_t* H, uint64_t m, const ShuffleScratch& s,
                                uint32_t* perm, cudaStream_t st) {
  if (m == 0) return;
  if (m == 1) {
    LGD_CUDA(cudaMemsetAsync(perm, 0, sizeof(uint32_t), st));
    return;
  }
  const uint64_t n = m - 1;
  keys_kernel<<<ceil_div(n, kThreads), kThreads, 0, st>>>(H, m, s.keys_in, s.vals_in);
  LGD_LAUNCH_CHECK();
  size_t bytes = s.sort_temp_bytes;
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(s.sort_temp, bytes, s.keys_in, s.keys_out, s.vals_in,
                                           s.vals_out, (int64_t)n, 0, bits_for(m), st));
  LGD_CUDA(cudaMemsetAsync(s.ptr, 0xff, m * sizeof(uint32_t), st));
  head_kernel<<<ceil_div(n, kThreads), kThreads, 0, st>>>(s.keys_out, s.vals_out, n, (uint32_t)m,
                                                          s.ptr);
  LGD_LAUNCH_CHECK();
  chase_kernel<<<ceil_div(m, kThreads), kThreads, 0, st>>>(s.ptr, m, s.G);
  LGD_LAUNCH_CHECK();
  final_kernel<<<ceil_div(n, kThreads), kThreads, 0, st>>>(s.keys_out, s.vals_out, n,
                                                           (uint32_t)m, s.G, perm);
  LGD_LAUNCH_CHECK();
  zero_kernel<<<1, 1, 0, st>>>(s.G, perm);
  LGD_LAUNCH_CHECK();
}

void launch_gather_edges(const uint32_t* edges, const uint32_t* perm, uint64_t m, uint32_t* out,
                         cudaStream_t st) {
  if (m == 0) return;
  gather_edges_kernel<<<ceil_div(m, kThreads), kThreads, 0, st>>>(edges, perm, m, out);
  LGD_LAUNCH_CHECK();
}

}  // namespace lgd
