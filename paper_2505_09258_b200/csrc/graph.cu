// graph.cu -- device side of the graph loader: the bucket index of
// make_partition_plan (graph.cpp:120-150) as a stable radix sort of bucket
// ids, the gather of edges into bucket order, and the synthetic power-law
// generator used for the benchmark shapes.
#include "common.cuh"
#include "detmath.cuh"
#include "internal.hpp"
#include "rng.cuh"

namespace lgd {

namespace {

constexpr int kThreads = 256;

__global__ void bucket_keys_kernel(const uint32_t* __restrict__ edges, uint64_t E, uint64_t stride,
                                   uint32_t n, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ iota,
                                   unsigned long long* __restrict__ counts) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const uint32_t b = (uint32_t)((edges[3 * e] / stride) * n + edges[3 * e + 2] / stride);
  keys[e] = b;
  iota[e] = (uint32_t)e;
  atomicAdd(counts + b, 1ull);
}

__global__ void gather3_kernel(const uint32_t* __restrict__ edges, const uint32_t* __restrict__ order,
                               uint64_t E, uint32_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const uint64_t s = order[i];
  out[3 * i] = edges[3 * s];
  out[3 * i + 1] = edges[3 * s + 1];
  out[3 * i + 2] = edges[3 * s + 2];
}

// Counter-based generator: edge e draws three splitmix64 words.  Endpoint
// ranks x in [1, V] follow a continuous Zipf law with density ~ x^-beta,
// beta = 1 / (alpha - 1) for degree exponent alpha (inverse CDF
// x = (1 + u (V^(1-beta) - 1))^(1/(1-beta))); alpha = 2.3 gives the top node
// ~0.3% of all endpoints, about Twitter's largest in-degree share.  Ranks are
// scattered over ids by a multiplicative permutation mod V so hubs land in
// every partition.  Relations are uniform over [0, R).  pow() is det_pow
// (detmath.cuh): IEEE-exact operations only, so the host restatement
// (oracle/legend_oracle.c: lo_powerlaw_edges) reproduces every edge.
__global__ void powerlaw_kernel(uint64_t V, uint64_t R, uint64_t E, double inv_one_minus_beta,
                                uint64_t mult, uint64_t seed, uint32_t* __restrict__ edges) {
  const double span = det_pow((double)V, 1.0 / inv_one_minus_beta) - 1.0;
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  uint64_t s = seed ^ (e * 0xd1342543de82ef95ull);
  const uint64_t a = splitmix64(s), b = splitmix64(s), c = splitmix64(s);
  auto endpoint = [&](uint64_t r) -> uint32_t {
    const double u = (double)(r >> 11) * 0x1.0p-53;
    uint64_t rank = (uint64_t)det_pow(1.0 + u * span, inv_one_minus_beta) - 1;
    if (rank >= V) rank = V - 1;
    // (rank * mult) mod V without overflow: 128-bit product
    const uint64_t lo = rank * mult;
    const uint64_t hi = __umul64hi(rank, mult);
    // reduce (hi:lo) mod V by long division in 2^32 steps (V < 2^63)
    uint64_t rem = hi % V;
    rem = ((rem << 32) | (lo >> 32)) % V;
    rem = ((rem << 32) | (lo & 0xffffffffull)) % V;
    return (uint32_t)rem;
  };
  edges[3 * e] = endpoint(a);
  edges[3 * e + 1] = R ? (uint32_t)(b % R) : 0xffffffffu;
  edges[3 * e + 2] = endpoint(c);
}

}  // namespace

void launch_bucket_keys(const uint32_t* edges, uint64_t E, uint64_t stride, uint32_t n,
                        uint32_t* keys, uint32_t* iota, unsigned long long* counts,
                        cudaStream_t st) {
  if (!E) return;
  bucket_keys_kernel<<<ceil_div(E, kThreads), kThreads, 0, st>>>(edges, E, stride, n, keys, iota,
                                                                 counts);
  LGD_LAUNCH_CHECK();
}

void launch_gather_u32x3(const uint32_t* edges, const uint32_t* order, uint64_t E, uint32_t* out,
                         cudaStream_t st) {
  if (!E) return;
  gather3_kernel<<<ceil_div(E, kThreads), kThreads, 0, st>>>(edges, order, E, out);
  LGD_LAUNCH_CHECK();
}

void launch_generate_powerlaw(uint64_t V, uint64_t R, uint64_t E, double alpha, uint64_t seed,
                              uint32_t* edges, cudaStream_t st) {
  if (!E) return;
  if (!(alpha > 2.0)) throw std::invalid_argument("power-law degree exponent must exceed 2");
  const double beta = 1.0 / (alpha - 1.0);
  // multiplier coprime with V (V < 2^32): walk odd candidates from a large prime
  uint64_t mult = 2654435761ull % V;
  auto gcd = [](uint64_t x, uint64_t y) {
    while (y) {
      const uint64_t t = x % y;
      x = y;
      y = t;
    }
    return x;
  };
  if (mult == 0) mult = 1;
  while (gcd(mult, V) != 1) mult = (mult + 1) % V ? (mult + 1) % V : 1;
  powerlaw_kernel<<<ceil_div(E, kThreads), kThreads, 0, st>>>(V, R, E, 1.0 / (1.0 - beta), mult,
                                                              seed, edges);
  LGD_LAUNCH_CHECK();
}

}  // namespace lgd
