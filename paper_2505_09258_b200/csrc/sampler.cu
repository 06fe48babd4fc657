// sampler.cu -- K2: the reference's sequential xoshiro256** consumers
// (sample_negatives train.cpp:365-373, the bucket shuffle's draws
// pipeline.cpp:297-301, store init store.cpp:19-25) as parallel chunked draws.
//
// Every lane owns a contiguous chunk of kChunk consumers.  A warp reaches its
// first stream position with a warp-cooperative GF(2) jump, then walks its 32
// lane origins with one jump-by-kChunk matrix each.  A draw that the
// reference would reject (r < (2^64 - b) % b, rng.hpp:43-46) is recorded with
// atomicMin; the fix-up kernel then regenerates everything from that consumer
// on, sequentially and exactly.  Rejections have probability < b/2^64 per
// draw, so the fix-up is a no-op in practice, but the result is bit-exact
// either way.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.hpp"
#include "rng.cuh"

namespace lgd {

namespace {

constexpr int kLog2Chunk = 7;
constexpr uint64_t kChunk = 1ull << kLog2Chunk;
constexpr int kThreads = 256;

// ------------------------------------------------------- jump tables (host)
void step_state(uint64_t s[4]) {  // the linear part of rng.hpp:25-31
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
}

void apply_host(const uint64_t* M, const uint64_t x[4], uint64_t y[4]) {
  y[0] = y[1] = y[2] = y[3] = 0;
  for (int c = 0; c < 256; ++c) {
    if ((x[c >> 6] >> (c & 63)) & 1) {
      for (int w = 0; w < 4; ++w) y[w] ^= M[c * 4 + w];
    }
  }
}

const std::vector<uint64_t>& host_tables() {
  static std::vector<uint64_t> tab;
  static std::once_flag once;
  std::call_once(once, [] {
    tab.assign(64 * 1024, 0);
    for (int c = 0; c < 256; ++c) {  // J[0] = M: column c = step(e_c)
      uint64_t s[4] = {0, 0, 0, 0};
      s[c >> 6] = 1ull << (c & 63);
      step_state(s);
      for (int w = 0; w < 4; ++w) tab[c * 4 + w] = s[w];
    }
    for (int i = 1; i < 64; ++i) {  // J[i] = J[i-1]^2
      const uint64_t* P = tab.data() + (size_t)(i - 1) * 1024;
      uint64_t* Q = tab.data() + (size_t)i * 1024;
      for (int c = 0; c < 256; ++c) apply_host(P, P + c * 4, Q + c * 4);
    }
  });
  return tab;
}

// --------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t pool_map(const Pool& p, uint64_t idx) {
  if (idx < p.end_index[0]) return (uint32_t)(p.first[0] + idx);
  if (p.n > 1 && idx < p.end_index[1]) return (uint32_t)(p.first[1] + (idx - p.end_index[0]));
  return (uint32_t)(p.first[2] + (idx - p.end_index[1]));
}

// Origin state of lane `lane`'s chunk for a warp whose first consumer is
// warp_first: all lanes return their own chunk origin.
__device__ __forceinline__ Xo lane_origin(const uint64_t* __restrict__ J, const Xo& s0,
                                          uint64_t first_raw, int lanes_needed, int lane) {
  Xo x = xo_jump_warp(J, s0, first_raw, lane);
  Xo mine = x;
  for (int l = 1; l < lanes_needed; ++l) {
    x = xo_apply_warp(J, kLog2Chunk, x, lane);
    if (lane == l) mine = x;
  }
  return mine;
}

enum Mode { kNodes = 0, kU64 = 1 };

template <int MODE>
__global__ void __launch_bounds__(kThreads) draw_const_kernel(
    const uint64_t* __restrict__ J, Xo s0, const uint64_t* __restrict__ d_pos, uint64_t count,
    Below bd, Pool pool, void* __restrict__ out, unsigned long long* __restrict__ d_reject) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const uint64_t warp_first = warp * 32 * kChunk;
  if (warp_first >= count) return;
  const uint64_t left = count - warp_first;
  const int lanes_needed = left >= 32 * kChunk ? 32 : (int)((left + kChunk - 1) / kChunk);
  const uint64_t base = d_pos ? *d_pos : 0;
  Xo x = lane_origin(J, s0, base + warp_first, lanes_needed, lane);
  const uint64_t q0 = warp_first + (uint64_t)lane * kChunk;
  if (lane >= lanes_needed) return;
  const uint64_t q1 = min(q0 + kChunk, count);
  uint64_t first_reject = ~0ull;
  for (uint64_t q = q0; q < q1; ++q) {
    const uint64_t r = xo_next(x);
    if (r < bd.threshold && first_reject == ~0ull) first_reject = q;
    const uint64_t v = mod_below(r, bd);
    if (MODE == kNodes) {
      static_cast<uint32_t*>(out)[q] = pool_map(pool, v);
    } else {
      static_cast<uint64_t*>(out)[q] = v;
    }
  }
  if (first_reject != ~0ull) atomicMin(d_reject, (unsigned long long)first_reject);
}

template <int MODE>
__global__ void draw_const_fixup(const uint64_t* __restrict__ J, Xo s0, uint64_t* d_pos,
                                 uint64_t count, Below bd, Pool pool, void* __restrict__ out,
                                 unsigned long long* d_reject) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint64_t base = d_pos ? *d_pos : 0;
  const uint64_t q0 = *d_reject;
  uint64_t used = count;
  if (q0 != ~0ull) {
    Xo x = xo_jump_thread(J, s0, base + q0);
    uint64_t raw = q0;
    for (uint64_t q = q0; q < count; ++q) {
      for (;;) {
        const uint64_t r = xo_next(x);
        ++raw;
        if (r >= bd.threshold) {
          const uint64_t v = r % bd.bound;
          if (MODE == kNodes) {
            static_cast<uint32_t*>(out)[q] = pool_map(pool, v);
          } else {
            static_cast<uint64_t*>(out)[q] = v;
          }
          break;
        }
      }
    }
    used = raw;
    *d_reject = ~0ull;
  }
  if (d_pos) *d_pos = base + used;
}

// Shuffle draws: consumer q (0 <= q < m-1) is next_below(m - q) and lands in
// H[m-1-q].  Bounds vary per draw, so the reduction is a plain 64-bit modulo.
__device__ __forceinline__ bool shuffle_rejects(uint64_t r, uint64_t b) {
  if (r >= b) return false;  // threshold = 2^64 mod b < b
  return r < (0 - b) % b;
}

__global__ void __launch_bounds__(kThreads) shuffle_draw_kernel(
    const uint64_t* __restrict__ J, Xo s0, const uint64_t* __restrict__ d_pos, uint64_t m,
    uint32_t* __restrict__ H, unsigned long long* __restrict__ d_reject) {
  const uint64_t count = m - 1;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const uint64_t warp_first = warp * 32 * kChunk;
  if (warp_first >= count) return;
  const uint64_t left = count - warp_first;
  const int lanes_needed = left >= 32 * kChunk ? 32 : (int)((left + kChunk - 1) / kChunk);
  const uint64_t base = d_pos ? *d_pos : 0;
  Xo x = lane_origin(J, s0, base + warp_first, lanes_needed, lane);
  const uint64_t q0 = warp_first + (uint64_t)lane * kChunk;
  if (lane >= lanes_needed) return;
  const uint64_t q1 = min(q0 + kChunk, count);
  uint64_t first_reject = ~0ull;
  for (uint64_t q = q0; q < q1; ++q) {
    const uint64_t r = xo_next(x);
    const uint64_t b = m - q;
    if (first_reject == ~0ull && shuffle_rejects(r, b)) first_reject = q;
    H[m - 1 - q] = (uint32_t)(r % b);
  }
  if (first_reject != ~0ull) atomicMin(d_reject, (unsigned long long)first_reject);
}

__global__ void shuffle_draw_fixup(const uint64_t* __restrict__ J, Xo s0, uint64_t* d_pos,
                                   uint64_t m, uint32_t* __restrict__ H,
                                   unsigned long long* d_reject) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint64_t count = m - 1;
  const uint64_t base = d_pos ? *d_pos : 0;
  const uint64_t q0 = *d_reject;
  uint64_t used = count;
  if (q0 != ~0ull) {
    Xo x = xo_jump_thread(J, s0, base + q0);
    uint64_t raw = q0;
    for (uint64_t q = q0; q < count; ++q) {
      const uint64_t b = m - q;
      const uint64_t th = (0 - b) % b;
      for (;;) {
        const uint64_t r = xo_next(x);
        ++raw;
        if (r >= th) {
          H[m - 1 - q] = (uint32_t)(r % b);
          break;
        }
      }
    }
    used = raw;
    *d_reject = ~0ull;
  }
  H[0] = 0;
  if (d_pos) *d_pos = base + used;
}

// store.cpp:19-25 / rng.hpp:36-39: v = f32(lo + (hi - lo) * ((r >> 11) * 2^-53)).
// Built with -fmad=false so the double expression rounds exactly like the
// reference (no contraction into an FMA).
__global__ void __launch_bounds__(kThreads) init_uniform_kernel(const uint64_t* __restrict__ J,
                                                                 Xo s0, uint64_t count, double lo,
                                                                 double span,
                                                                 float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const uint64_t warp_first = warp * 32 * kChunk;
  if (warp_first >= count) return;
  const uint64_t left = count - warp_first;
  const int lanes_needed = left >= 32 * kChunk ? 32 : (int)((left + kChunk - 1) / kChunk);
  Xo x = lane_origin(J, s0, warp_first, lanes_needed, lane);
  const uint64_t q0 = warp_first + (uint64_t)lane * kChunk;
  if (lane >= lanes_needed) return;
  const uint64_t q1 = min(q0 + kChunk, count);
  for (uint64_t q = q0; q < q1; ++q) {
    const uint64_t r = xo_next(x);
    const double u = (double)(r >> 11) * 0x1.0p-53;
    out[q] = (float)(lo + span * u);
  }
}

unsigned grid_for(uint64_t count) {
  const uint64_t per_block = (uint64_t)(kThreads / 32) * 32 * kChunk;
  return ceil_div(count ? count : 1, per_block);
}

}  // namespace

void host_jump(Xo& x, uint64_t n) {
  const auto& tab = host_tables();
  for (int m = 0; n; ++m, n >>= 1) {
    if (n & 1) {
      uint64_t y[4];
      apply_host(tab.data() + (size_t)m * 1024, x.s, y);
      std::memcpy(x.s, y, sizeof y);
    }
  }
}

const uint64_t* jump_tables(int device) {
  static std::mutex mu;
  static std::vector<uint64_t*> per_device;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)per_device.size() <= device) per_device.resize(device + 1, nullptr);
  if (!per_device[device]) {
    const auto& tab = host_tables();
    uint64_t* d = nullptr;
    LGD_CUDA(cudaMalloc(&d, tab.size() * sizeof(uint64_t)));
    LGD_CUDA(cudaMemcpy(d, tab.data(), tab.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    per_device[device] = d;
  }
  return per_device[device];
}

static const uint64_t* current_tables() {
  int dev = 0;
  LGD_CUDA(cudaGetDevice(&dev));
  return jump_tables(dev);
}

void launch_sample_nodes(const StreamSlot& s, uint64_t count, const Pool& pool, uint32_t* out,
                         cudaStream_t st) {
  if (count == 0) return;
  const uint64_t* J = current_tables();
  const Below bd = make_below(pool.end_index[pool.n - 1]);
  draw_const_kernel<kNodes><<<grid_for(count), kThreads, 0, st>>>(J, s.origin, s.d_pos, count, bd,
                                                                   pool, out, s.d_reject);
  LGD_LAUNCH_CHECK();
  draw_const_fixup<kNodes><<<1, 32, 0, st>>>(J, s.origin, s.d_pos, count, bd, pool, out,
                                              s.d_reject);
  LGD_LAUNCH_CHECK();
}

void launch_below_u64(const StreamSlot& s, uint64_t count, uint64_t bound, uint64_t* out,
                      cudaStream_t st) {
  if (count == 0) return;
  const uint64_t* J = current_tables();
  const Below bd = make_below(bound);
  Pool pool{};
  draw_const_kernel<kU64><<<grid_for(count), kThreads, 0, st>>>(J, s.origin, s.d_pos, count, bd,
                                                                 pool, out, s.d_reject);
  LGD_LAUNCH_CHECK();
  draw_const_fixup<kU64><<<1, 32, 0, st>>>(J, s.origin, s.d_pos, count, bd, pool, out,
                                            s.d_reject);
  LGD_LAUNCH_CHECK();
}

void launch_shuffle_draws(const StreamSlot& s, uint64_t m, uint32_t* H, cudaStream_t st) {
  if (m < 2) {
    if (m == 1) LGD_CUDA(cudaMemsetAsync(H, 0, sizeof(uint32_t), st));
    return;
  }
  const uint64_t* J = current_tables();
  shuffle_draw_kernel<<<grid_for(m - 1), kThreads, 0, st>>>(J, s.origin, s.d_pos, m, H,
                                                            s.d_reject);
  LGD_LAUNCH_CHECK();
  shuffle_draw_fixup<<<1, 32, 0, st>>>(J, s.origin, s.d_pos, m, H, s.d_reject);
  LGD_LAUNCH_CHECK();
}

void launch_init_uniform(const uint64_t* J, uint64_t seed, uint64_t count, uint32_t dim,
                         float* out, cudaStream_t st) {
  if (count == 0) return;
  const double bound = 0.5 / std::sqrt(static_cast<double>(dim));
  const double lo = -bound, hi = bound;
  init_uniform_kernel<<<grid_for(count), kThreads, 0, st>>>(J, xo_seed(seed), count, lo, hi - lo,
                                                            out);
  LGD_LAUNCH_CHECK();
}

}  // namespace lgd
