// rng.cuh -- the reference's xoshiro256** stream (rng.hpp:7-67), reproduced
// bit-exactly on the device, plus GF(2) jump-ahead so that any stream
// position can be reached in O(log offset) matrix-vector products.
//
// The xoshiro256** state update is linear over GF(2): s' = M s for a fixed
// 256x256 bit matrix M.  The host builds J[i] = M^(2^i), i < 64 (jump.cpp);
// the device applies the set bits of an offset.  A matrix is stored column
// major: column c (= M e_c, bit c of the state, word c/64) is 4 u64 words.
#pragma once

#include <cstdint>

namespace lgd {

struct Xo {
  uint64_t s[4];
};

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// Rng(seed) constructor state (rng.hpp:18-21)
__host__ __device__ __forceinline__ Xo xo_seed(uint64_t seed) {
  Xo x;
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) x.s[i] = splitmix64(s);
  return x;
}

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t v, int k) {
  return (v << k) | (v >> (64 - k));
}

// next_u64 (rng.hpp:23-33)
__host__ __device__ __forceinline__ uint64_t xo_next(Xo& x) {
  const uint64_t result = rotl64(x.s[1] * 5, 7) * 9;
  const uint64_t t = x.s[1] << 17;
  x.s[2] ^= x.s[0];
  x.s[3] ^= x.s[1];
  x.s[1] ^= x.s[2];
  x.s[0] ^= x.s[3];
  x.s[2] ^= t;
  x.s[3] = rotl64(x.s[3], 45);
  return result;
}

// derive_seed (rng.hpp:57-67)
__host__ __device__ __forceinline__ uint64_t derive_seed(uint64_t base, uint64_t a, uint64_t b = 0,
                                                         uint64_t c = 0) {
  uint64_t s = base;
  splitmix64(s);
  s ^= 0x516cc24f80775842ull + a;
  splitmix64(s);
  s ^= 0x2545f4914f6cdd1dull * (b + 1);
  splitmix64(s);
  s ^= 0x9e6c63d0876a9a47ull * (c + 1);
  return splitmix64(s);
}

constexpr uint64_t kTagBucket = 0x62756b74ull;    // "bukt"  pipeline.cpp:296
constexpr uint64_t kTagEval = 0x65766179ull;      // "evay"  train.cpp:399
constexpr uint64_t kTagRelations = 0x52454c53ull; // "RELS"  store.cpp:17

// ---------------------------------------------------------------- jumps
// J: 64 matrices x 256 columns x 4 words (512 KB), device resident.

// One thread applies J[m] to x.
__device__ __forceinline__ Xo xo_apply_thread(const uint64_t* __restrict__ J, int m, const Xo& x) {
  const ulonglong2* col = reinterpret_cast<const ulonglong2*>(J + (size_t)m * 1024);
  uint64_t y0 = 0, y1 = 0, y2 = 0, y3 = 0;
#pragma unroll 1
  for (int w = 0; w < 4; ++w) {
    uint64_t bits = x.s[w];
    while (bits) {
      const int b = __ffsll((long long)bits) - 1;
      bits &= bits - 1;
      const int c = w * 64 + b;
      const ulonglong2 lo = __ldg(col + 2 * c);
      const ulonglong2 hi = __ldg(col + 2 * c + 1);
      y0 ^= lo.x;
      y1 ^= lo.y;
      y2 ^= hi.x;
      y3 ^= hi.y;
    }
  }
  Xo y;
  y.s[0] = y0;
  y.s[1] = y1;
  y.s[2] = y2;
  y.s[3] = y3;
  return y;
}

// One thread jumps x forward by n draws.
__device__ __forceinline__ Xo xo_jump_thread(const uint64_t* __restrict__ J, Xo x, uint64_t n) {
  for (int m = 0; n; ++m, n >>= 1)
    if (n & 1) x = xo_apply_thread(J, m, x);
  return x;
}

// A whole warp applies J[m] to the (warp-uniform) x: lane l owns state bits
// [8l, 8l+8); the partial column sums are XOR-reduced across the warp.
__device__ __forceinline__ Xo xo_apply_warp(const uint64_t* __restrict__ J, int m, const Xo& x,
                                            int lane) {
  const ulonglong2* col = reinterpret_cast<const ulonglong2*>(J + (size_t)m * 1024);
  const int w = lane >> 3;
  const int sh = (lane & 7) * 8;
  uint32_t bits = (uint32_t)((x.s[w] >> sh) & 0xffu);
  uint64_t y0 = 0, y1 = 0, y2 = 0, y3 = 0;
  while (bits) {
    const int b = __ffs(bits) - 1;
    bits &= bits - 1;
    const int c = lane * 8 + b;
    const ulonglong2 lo = __ldg(col + 2 * c);
    const ulonglong2 hi = __ldg(col + 2 * c + 1);
    y0 ^= lo.x;
    y1 ^= lo.y;
    y2 ^= hi.x;
    y3 ^= hi.y;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    y0 ^= __shfl_xor_sync(0xffffffffu, y0, off);
    y1 ^= __shfl_xor_sync(0xffffffffu, y1, off);
    y2 ^= __shfl_xor_sync(0xffffffffu, y2, off);
    y3 ^= __shfl_xor_sync(0xffffffffu, y3, off);
  }
  Xo y;
  y.s[0] = y0;
  y.s[1] = y1;
  y.s[2] = y2;
  y.s[3] = y3;
  return y;
}

// The whole warp jumps the warp-uniform x forward by the warp-uniform n.
__device__ __forceinline__ Xo xo_jump_warp(const uint64_t* __restrict__ J, Xo x, uint64_t n,
                                           int lane) {
  for (int m = 0; n; ++m, n >>= 1)
    if (n & 1) x = xo_apply_warp(J, m, x, lane);
  return x;
}

// --------------------------------------------------------- next_below
// r % b for 64-bit r, b via a precomputed reciprocal: q = mulhi(r, inv) with
// inv = floor((2^64 - 1) / b) underestimates floor(r / b) by at most 1, so
// one conditional subtraction finishes the reduction exactly.
struct Below {
  uint64_t bound;
  uint64_t threshold;  // (2^64 - bound) % bound: draws below it are rejected
  uint64_t inv;
};

__host__ __device__ __forceinline__ Below make_below(uint64_t bound) {
  Below b;
  b.bound = bound;
  b.threshold = (0 - bound) % bound;
  b.inv = ~0ull / bound;
  return b;
}

__device__ __forceinline__ uint64_t mod_below(uint64_t r, const Below& b) {
  const uint64_t q = __umul64hi(r, b.inv);
  uint64_t rem = r - q * b.bound;
  if (rem >= b.bound) rem -= b.bound;
  return rem;
}

}  // namespace lgd
