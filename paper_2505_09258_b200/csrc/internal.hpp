// internal.hpp -- launchers shared between the CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rng.cuh"

namespace lgd {

// ------------------------------------------------------------ sampler.cu
// Jump tables J[i] = M^(2^i) for the xoshiro256** state update, uploaded once
// per device (512 KB).
const uint64_t* jump_tables(int device);
void host_jump(Xo& x, uint64_t n);  // host reference of the device jump (tests)

// Resident sampling pool: up to 3 node ranges, ascending first node
// (ResidentTable entries_, train.cpp:112-119, 190-202).
struct Pool {
  uint64_t first[3];
  uint64_t end_index[3];  // inclusive prefix of counts
  int n;
};

// Stream bookkeeping for one Rng: origin state, device offset counter and a
// device "first rejected consumer" slot (UINT64_MAX when none).
struct StreamSlot {
  Xo origin;
  uint64_t* d_pos;        // raw draws consumed so far
  unsigned long long* d_reject;
};

// next_below(pool total) x count, mapped through the pool, written as u32 node
// ids; advances *d_pos by count + rejections.  Two launches: a parallel draw
// and a one-thread fix-up that re-runs the tail sequentially only if some
// draw was rejected (probability < bound / 2^64 per draw).
void launch_sample_nodes(const StreamSlot& s, uint64_t count, const Pool& pool, uint32_t* out,
                         cudaStream_t st);
// next_below(bound) x count as raw u64 values (primitive tests).
void launch_below_u64(const StreamSlot& s, uint64_t count, uint64_t bound, uint64_t* out,
                      cudaStream_t st);
// The m-1 Fisher-Yates draws of pipeline.cpp:297-301: H[t] = next_below(t+1)
// for t = m-1 down to 1 (draw order), H[0] = 0.
void launch_shuffle_draws(const StreamSlot& s, uint64_t m, uint32_t* H, cudaStream_t st);
// fill_uniform_rows (store.cpp:19-25): count f32 values of Rng(seed).
void launch_init_uniform(const uint64_t* J, uint64_t seed, uint64_t count, uint32_t dim,
                         float* out, cudaStream_t st);

// ------------------------------------------------------------ shuffle.cu
struct ShuffleScratch {
  uint32_t* keys_in;
  uint32_t* vals_in;
  uint32_t* keys_out;
  uint32_t* vals_out;
  uint32_t* ptr;
  uint32_t* G;
  void* sort_temp;
  size_t sort_temp_bytes;
};
size_t shuffle_sort_temp_bytes(uint64_t m_max);
// perm[i] = original position of the element that ends at position i after
// the sequential swaps "for t = m-1..1: swap(A[t], A[H[t]])".
void launch_shuffle_permutation(const uint32_t* H, uint64_t m, const ShuffleScratch& s,
                                uint32_t* perm, cudaStream_t st);
// out[i] = edges[perm[i]] (12-byte records); perm may be null (identity).
void launch_gather_edges(const uint32_t* edges, const uint32_t* perm, uint64_t m, uint32_t* out,
                         cudaStream_t st);

// -------------------------------------------------------------- graph.cu
void launch_bucket_keys(const uint32_t* edges, uint64_t E, uint64_t stride, uint32_t n,
                        uint32_t* keys, uint32_t* iota, unsigned long long* counts,
                        cudaStream_t st);
void launch_gather_u32x3(const uint32_t* edges, const uint32_t* order, uint64_t E, uint32_t* out,
                         cudaStream_t st);
void launch_generate_powerlaw(uint64_t V, uint64_t R, uint64_t E, double zipf, uint64_t seed,
                              uint32_t* edges, cudaStream_t st);

}  // namespace lgd
