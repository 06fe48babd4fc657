// evaluate.cu -- K6: evaluate() (train.cpp:375-412) on the device.
// Candidates: one thread per test edge replays that edge's own stream
// Rng(derive_seed(seed, "evay", t)) sequentially (999 draws), so rejections
// are handled exactly as in the reference.  Scoring: one warp per test edge,
// FP64 dot products against the true destination and every candidate,
// pessimistic ties (rank = 1 + #{score >= true score}).
#include "common.cuh"
#include "evaluate.cuh"
#include "rng.cuh"

namespace lgd {

namespace {

__global__ void eval_candidates_kernel(uint64_t seed, uint64_t T, uint32_t ncand, uint64_t V,
                                       uint32_t* __restrict__ cand) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  Xo x = xo_seed(derive_seed(seed, kTagEval, t));
  const Below bd = make_below(V);
  for (uint32_t c = 0; c < ncand; ++c) {
    uint64_t r;
    do {
      r = xo_next(x);
    } while (r < bd.threshold);
    cand[t * ncand + c] = (uint32_t)(r % V);
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// ir1 held as up to 16 doubles per lane: element i = lane + 32 c.
template <int NC>
__global__ void eval_score_kernel(int kind, uint32_t d, const float* __restrict__ theta,
                                  const float* __restrict__ rel, const uint32_t* __restrict__ edges,
                                  uint64_t T, uint32_t ncand, const uint32_t* __restrict__ cand,
                                  uint32_t hits_k, double* __restrict__ rr,
                                  double* __restrict__ hit) {
  const int lane = threadIdx.x & 31;
  const uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= T) return;
  const uint32_t s = edges[3 * t], r = edges[3 * t + 1], dd = edges[3 * t + 2];
  const uint32_t h = d / 2;
  double x[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint32_t i = lane + 32 * c;
    x[c] = 0.0;
    if (i >= d) continue;
    const float* sr = theta + (size_t)s * d;
    if (kind == 0) {
      x[c] = sr[i];
    } else if (kind == 1) {
      x[c] = (double)sr[i] * (double)rel[(size_t)r * d + i];
    } else if (kind == 3) {
      x[c] = (double)sr[i] + (double)rel[(size_t)r * d + i];
    } else {
      const float* rl = rel + (size_t)r * d;
      const uint32_t j = i < h ? i : i - h;
      const double a = sr[j], b = sr[j + h], p = rl[j], q = rl[j + h];
      x[c] = i < h ? a * p - b * q : a * q + b * p;
    }
  }
  auto score = [&](uint32_t node) {
    const float* row = theta + (size_t)node * d;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t i = lane + 32 * c;
      if (i < d) {
        if (kind == 3) {
          const double q = x[c] - (double)row[i];
          acc += q * q;
        } else {
          acc += x[c] * (double)row[i];
        }
      }
    }
    return kind == 3 ? -sqrt(warp_sum(acc)) : warp_sum(acc);
  };
  const double truth = score(dd);
  uint32_t beaten = 0;
  for (uint32_t c = 0; c < ncand; ++c)
    if (score(cand[t * ncand + c]) >= truth) ++beaten;
  if (lane == 0) {
    const uint64_t rank = 1ull + beaten;
    rr[t] = 1.0 / (double)rank;
    hit[t] = rank <= hits_k ? 1.0 : 0.0;
  }
}

__global__ void mean_kernel(const double* __restrict__ v, uint64_t n, double* out) {
  __shared__ double part[1024];
  double s = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += 1024) s += v[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0] / (double)n;
}

}  // namespace

void launch_evaluate(const EvalArgs& a, cudaStream_t st) {
  eval_candidates_kernel<<<ceil_div(a.T, 128), 128, 0, st>>>(a.seed, a.T, a.ncand, a.V, a.cand);
  LGD_LAUNCH_CHECK();
  const unsigned grid = ceil_div(a.T * 32, 256);
  const uint32_t nc = (a.dim + 31) / 32;
#define LGD_EVAL(NC)                                                                        \
  eval_score_kernel<NC><<<grid, 256, 0, st>>>(a.kind, a.dim, a.theta, a.rel, a.edges, a.T, \
                                              a.ncand, a.cand, a.hits_k, a.rr, a.hit)
  if (nc <= 1) {
    LGD_EVAL(1);
  } else if (nc <= 2) {
    LGD_EVAL(2);
  } else if (nc <= 4) {
    LGD_EVAL(4);
  } else if (nc <= 8) {
    LGD_EVAL(8);
  } else {
    LGD_EVAL(16);
  }
#undef LGD_EVAL
  LGD_LAUNCH_CHECK();
  mean_kernel<<<1, 1024, 0, st>>>(a.rr, a.T, a.out);
  LGD_LAUNCH_CHECK();
  mean_kernel<<<1, 1024, 0, st>>>(a.hit, a.T, a.out + 1);
  LGD_LAUNCH_CHECK();
}

}  // namespace lgd
