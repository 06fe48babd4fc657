// train.cu -- the per-batch hot path: batch_loss + batch_gradients +
// adagrad_step (train.cpp:217-363) as
//   K3 score_kernel    warp per positive; the 2+k+t embedding rows are pulled
//                      into shared memory by TMA bulk copies
//                      (cp.async.bulk, one per row, mbarrier-tracked, double
//                      buffered across the warp's positives); FP64 math
//                      exactly as the reference orders it per element,
//                      warp-shuffle reductions for the dot products.
//   sort               CUB onesweep radix sort of the P(k+2) contribution
//                      node ids (stable, so each node's contributions stay in
//                      the reference's std::map visit order: positive
//                      ascending, then dst, negatives j ascending, src).
//   K4 segment passes  warp per 32 sorted contributions: sum each node's
//                      contributions in order (FP64), then one Adagrad row
//                      update (train.cpp:342-354) per unique node -- a
//                      sort-by-node segmented reduction, no atomics on rows.
//                      Segments that cross a 32-item chunk are finished by a
//                      second pass from per-chunk partial sums.
//   relation path      the same segmented reduction over relation ids.
// All FP64 expressions are compiled with -fmad=false so products and sums
// round exactly like the reference's unfused x86-64 double arithmetic.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "train.cuh"

namespace lgd {

namespace {

constexpr int kScoreWarps = 4;
constexpr int kSegThreads = 256;
constexpr uint8_t kNoHead = 1;
constexpr uint8_t kContOut = 2;

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

// 1-D TMA: global -> shared, completion counted on the mbarrier in bytes.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// --------------------------------------------------- lane element mapping
// Dot / DistMult: lane owns elements lane + 32c (c < NC).
// ComplEx (half-split encoding, train.hpp:17-18): lane owns real index
// j = lane + 32c and its imaginary partner j + h; slots c (re) and NC + c (im).
template <int KIND, int NC>
struct Map {
  static constexpr int NE = KIND == 2 ? 2 * NC : NC;
  __device__ __forceinline__ static int idx(int e, int lane, uint32_t h) {
    if (KIND == 2) return e < NC ? lane + 32 * e : lane + 32 * (e - NC) + (int)h;
    return lane + 32 * e;
  }
  __device__ __forceinline__ static bool ok(int e, int lane, uint32_t d, uint32_t h) {
    if (KIND == 2) return lane + 32 * (e < NC ? e : e - NC) < (int)h;
    return lane + 32 * e < (int)d;
  }
};

// IR1 = s (x) r (combine_src_rel, train.cpp:39-60) for the lane's elements.
template <int KIND, int NC>
__device__ __forceinline__ void combine(const float* s, const float* r, int lane, uint32_t d,
                                        uint32_t h, double* x) {
  using M = Map<KIND, NC>;
  if (KIND == 2) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      x[c] = 0.0;
      x[c + NC] = 0.0;
      if (M::ok(c, lane, d, h)) {
        const int j = lane + 32 * c;
        const double sr = s[j], si = s[j + h];
        const double rr = r[j], ri = r[j + h];
        x[c] = sr * rr - si * ri;
        x[c + NC] = sr * ri + si * rr;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < NC; ++e) {
      x[e] = 0.0;
      if (M::ok(e, lane, d, h)) {
        const int i = lane + 32 * e;
        x[e] = KIND == 0 ? (double)s[i] : (double)s[i] * (double)r[i];
      }
    }
  }
}

// g += adj_other(mix) (adjoint_combine, train.cpp:65-85) for the lane's elements.
template <int KIND, int NC>
__device__ __forceinline__ void adjoint_add(const float* other, const double* mixrow, int lane,
                                            uint32_t d, uint32_t h, double* g) {
  using M = Map<KIND, NC>;
  if (KIND == 2) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (M::ok(c, lane, d, h)) {
        const int j = lane + 32 * c;
        const double orr = other[j], ori = other[j + h];
        const double mr = mixrow[j], mi = mixrow[j + h];
        g[c] += orr * mr + ori * mi;
        g[c + NC] += orr * mi - ori * mr;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < NC; ++e) {
      if (M::ok(e, lane, d, h)) {
        const int i = lane + 32 * e;
        if (KIND == 0) {
          g[e] += mixrow[i];
        } else {
          g[e] += (double)other[i] * mixrow[i];
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K3 score
// Shared memory per warp: 2 row buffers of (k+3) x dpad floats (src, rel,
// dst, k negatives), then f_j and e_j scratch (k doubles each).
template <int KIND, int NC, bool TMA>
__global__ void __launch_bounds__(kScoreWarps * 32) score_kernel(BatchArgs a, uint32_t dpad) {
  extern __shared__ __align__(128) unsigned char smem[];
  using M = Map<KIND, NC>;
  constexpr int NE = M::NE;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t k = a.k, d = a.dim, h = d / 2;
  const bool typed = KIND != 0;
  const uint32_t nrows = k + 3;
  const size_t buf_floats = (size_t)nrows * dpad;
  const size_t warp_bytes = 2 * buf_floats * sizeof(float) + 2 * (size_t)k * sizeof(double);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + 2 * warp;
  float* rows = reinterpret_cast<float*>(smem + 16 * kScoreWarps + warp * warp_bytes);
  double* fj = reinterpret_cast<double*>(rows + 2 * buf_floats);
  double* ej = fj + k;

  if (TMA) {
    if (lane == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  const uint32_t row_bytes = d * sizeof(float);
  const uint32_t tx_bytes = (typed ? nrows : nrows - 1) * row_bytes;

  auto issue = [&](uint64_t p, int b) {
    float* base = rows + b * buf_floats;
    const uint32_t s = a.edges[3 * p], r = a.edges[3 * p + 1], t = a.edges[3 * p + 2];
    if (TMA) {
      if (lane == 0) mbar_arrive_expect_tx(bars + b, tx_bytes);
      __syncwarp();
      for (uint32_t row = lane; row < nrows; row += 32) {
        const float* src;
        if (row == 0) {
          src = a.theta + (size_t)s * d;
        } else if (row == 1) {
          if (!typed) continue;
          src = a.rel_theta + (size_t)r * d;
        } else if (row == 2) {
          src = a.theta + (size_t)t * d;
        } else {
          src = a.theta + (size_t)a.negs[p * k + (row - 3)] * d;
        }
        bulk_g2s(base + row * dpad, src, row_bytes, bars + b);
      }
    } else {
      for (uint32_t row = 0; row < nrows; ++row) {
        const float* src;
        if (row == 0) {
          src = a.theta + (size_t)s * d;
        } else if (row == 1) {
          if (!typed) continue;
          src = a.rel_theta + (size_t)r * d;
        } else if (row == 2) {
          src = a.theta + (size_t)t * d;
        } else {
          src = a.theta + (size_t)a.negs[p * k + (row - 3)] * d;
        }
        for (uint32_t i = lane; i < d; i += 32) base[row * dpad + i] = src[i];
      }
    }
  };

  const uint64_t nwarps = (uint64_t)gridDim.x * kScoreWarps;
  uint64_t p = (uint64_t)blockIdx.x * kScoreWarps + warp;
  uint32_t phase0 = 0, phase1 = 0;
  int b = 0;
  if (p < a.P) issue(p, 0);
  for (; p < a.P; p += nwarps, b ^= 1) {
    const uint64_t pn = p + nwarps;
    if (pn < a.P) issue(pn, b ^ 1);
    if (TMA) {
      uint64_t* bar = bars + b;
      const uint32_t ph = b ? phase1 : phase0;
      while (!mbar_try_wait(bar, ph)) {
      }
      if (b) {
        phase1 ^= 1;
      } else {
        phase0 ^= 1;
      }
    }
    __syncwarp();
    const float* R = rows + b * buf_floats;
    const float* srow = R;
    const float* rrow = R + dpad;
    const float* drow = R + 2 * dpad;

    double x[NE];
    combine<KIND, NC>(srow, rrow, lane, d, h, x);
    // positive score (train.cpp:246-252)
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (M::ok(e, lane, d, h)) acc += x[e] * (double)drow[M::idx(e, lane, h)];
    const double pos = warp_sum(acc);
    // negative scores (train.cpp:256-264)
    for (uint32_t j = 0; j < k; ++j) {
      const float* nrow = R + (3 + j) * dpad;
      double f = 0.0;
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (M::ok(e, lane, d, h)) f += x[e] * (double)nrow[M::idx(e, lane, h)];
      f = warp_sum(f);
      if (lane == (int)(j & 31)) fj[j] = f;
    }
    __syncwarp();
    double row_max = -INFINITY;
    for (uint32_t j = 0; j < k; ++j) {
      const double f = fj[j];
      row_max = row_max < f ? f : row_max;  // std::max(row_max, f)
    }
    for (uint32_t j = lane; j < k; j += 32) ej[j] = exp(fj[j] - row_max);  // IR3
    __syncwarp();
    double sum = 0.0;
    for (uint32_t j = 0; j < k; ++j) sum += ej[j];  // sequential j, every lane
    const double inv_sum = 1.0 / sum;
    for (uint32_t j = lane; j < k; j += 32) a.w[p * k + j] = ej[j] * inv_sum;
    if (lane == 0) a.loss[p] = -(pos - (row_max + log(sum)));  // train.cpp:274

    // mix = sum_j w_j neg_j - dst (train.cpp:306-323)
    double mx[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e)
      mx[e] = M::ok(e, lane, d, h) ? -(double)drow[M::idx(e, lane, h)] : 0.0;
    for (uint32_t j = 0; j < k; ++j) {
      const float* nrow = R + (3 + j) * dpad;
      const double w = ej[j] * inv_sum;
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (M::ok(e, lane, d, h)) mx[e] += w * (double)nrow[M::idx(e, lane, h)];
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      if (M::ok(e, lane, d, h)) {
        const int i = M::idx(e, lane, h);
        a.mix[p * d + i] = mx[e];
        a.snap[p * d + i] = srow[i];
      }
    }
    // contribution keys in the reference's visit order: dst, negs, src
    const uint64_t kb = p * (k + 2);
    if (lane == 0) {
      a.node_keys[kb] = a.edges[3 * p + 2];
      a.node_keys[kb + k + 1] = a.edges[3 * p];
      if (typed) a.rel_keys[p] = a.edges[3 * p + 1];
    }
    for (uint32_t j = lane; j < k; j += 32) a.node_keys[kb + 1 + j] = a.negs[p * k + j];
    __syncwarp();
  }
}

// --------------------------------------------------------- loss reduction
__global__ void __launch_bounds__(1024) loss_reduce_kernel(const double* __restrict__ loss,
                                                           uint64_t P, double* out) {
  __shared__ double part[1024];
  double s = 0.0;
  for (uint64_t i = threadIdx.x; i < P; i += 1024) s += loss[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

// ------------------------------------------------- K4 segmented reduction
// One item of the sorted contribution list, added to the lane's elements.
template <int KIND, int NC, bool REL>
__device__ __forceinline__ void add_item(const BatchArgs& a, uint32_t val, int lane, double* g) {
  using M = Map<KIND, NC>;
  const uint32_t d = a.dim, h = d / 2, k = a.k;
  if (REL) {  // relation gradient: adj_src(mix) (train.cpp:328-332)
    const uint64_t p = val;
    adjoint_add<KIND, NC>(a.snap + p * d, a.mix + p * d, lane, d, h, g);
    return;
  }
  const uint64_t p = val / (k + 2);
  const uint32_t slot = val - (uint32_t)(p * (k + 2));
  const float* rel = KIND != 0 ? a.rel_theta + (size_t)a.edges[3 * p + 1] * d : nullptr;
  if (slot <= k) {
    double x[M::NE];
    combine<KIND, NC>(a.snap + p * d, rel, lane, d, h, x);
    if (slot == 0) {  // dst: g -= IR1 (train.cpp:310)
#pragma unroll
      for (int e = 0; e < M::NE; ++e) g[e] -= x[e];
    } else {  // negative j: g += w_j IR1 (train.cpp:320)
      const double w = a.w[p * k + (slot - 1)];
#pragma unroll
      for (int e = 0; e < M::NE; ++e) g[e] += w * x[e];
    }
  } else {  // src: g += adj_rel(mix) (train.cpp:327)
    adjoint_add<KIND, NC>(rel, a.mix + p * d, lane, d, h, g);
  }
}

// adagrad_update (train.cpp:342-354) on one row, or the gradient itself in
// gradient-only mode.
template <int KIND, int NC, bool REL>
__device__ __forceinline__ void finish_row(const BatchArgs& a, uint32_t row, const double* g,
                                           int lane) {
  using M = Map<KIND, NC>;
  const uint32_t d = a.dim, h = d / 2;
  double* gout = REL ? a.grad_rels : a.grad_nodes;
  if (gout) {
#pragma unroll
    for (int e = 0; e < M::NE; ++e)
      if (M::ok(e, lane, d, h)) gout[(size_t)row * d + M::idx(e, lane, h)] = g[e];
    if (lane == 0) (REL ? a.grad_rel_flag : a.grad_node_flag)[row] = 1;
    return;
  }
  float* th = (REL ? a.rel_theta : a.theta) + (size_t)row * d;
  float* st = (REL ? a.rel_state : a.state) + (size_t)row * d;
  float tv[M::NE], sv[M::NE];
#pragma unroll
  for (int e = 0; e < M::NE; ++e) {
    if (M::ok(e, lane, d, h)) {
      const int i = M::idx(e, lane, h);
      tv[e] = th[i];
      sv[e] = st[i];
    }
  }
#pragma unroll
  for (int e = 0; e < M::NE; ++e) {
    if (M::ok(e, lane, d, h)) {
      const int i = M::idx(e, lane, h);
      const double gi = g[e];
      const double acc = (double)sv[e] + gi * gi;
      st[i] = (float)acc;
      th[i] = (float)((double)tv[e] - a.lr * gi / (sqrt(acc) + a.eps));
    }
  }
}

template <int KIND, int NC, bool REL>
__global__ void __launch_bounds__(kSegThreads) segment_pass1(BatchArgs a, uint64_t n,
                                                             const uint32_t* __restrict__ skeys,
                                                             const uint32_t* __restrict__ svals) {
  using M = Map<KIND, NC>;
  const int lane = threadIdx.x & 31;
  const uint64_t c = ((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5;
  const uint64_t base = c * 32;
  if (base >= n) return;
  const uint64_t end = min(base + 32, n);
  const uint64_t i = base + lane;
  const uint32_t key = i < n ? skeys[i] : 0;
  const bool head = i < n && (i == 0 || skeys[i - 1] != key);
  uint32_t mask = __ballot_sync(0xffffffffu, head);
  const bool cont_out = end < n && skeys[end] == skeys[end - 1];
  double* first_out = a.part_first + c * a.dim;
  double* last_out = a.part_last + c * a.dim;
  const uint32_t d = a.dim, h = d / 2;

  auto accumulate = [&](uint64_t from, uint64_t to, double* g) {
#pragma unroll
    for (int e = 0; e < M::NE; ++e) g[e] = 0.0;
    for (uint64_t q = from; q < to; ++q) add_item<KIND, NC, REL>(a, svals[q], lane, g);
  };
  auto store_partial = [&](double* dst, const double* g) {
#pragma unroll
    for (int e = 0; e < M::NE; ++e)
      if (M::ok(e, lane, d, h)) dst[M::idx(e, lane, h)] = g[e];
  };

  if (!(mask & 1u)) {  // leading piece continues a segment from the previous chunk
    const uint64_t to = mask ? base + (__ffs(mask) - 1) : end;
    double g[M::NE];
    accumulate(base, to, g);
    store_partial(first_out, g);
  }
  const uint32_t heads = __popc(mask);
  while (mask) {
    const int hb = __ffs(mask) - 1;
    mask &= mask - 1;
    const uint64_t from = base + hb;
    const uint64_t to = mask ? base + (__ffs(mask) - 1) : end;
    double g[M::NE];
    accumulate(from, to, g);
    if (to == end && cont_out) {
      store_partial(last_out, g);  // finished in pass 2
    } else {
      finish_row<KIND, NC, REL>(a, skeys[from], g, lane);
    }
  }
  if (lane == 0) {
    a.chunk_flags[c] = (heads ? 0 : kNoHead) | (cont_out ? kContOut : 0);
    if (heads) atomicAdd(a.counters + (REL ? 1 : 0), (unsigned long long)heads);
  }
}

template <int KIND, int NC, bool REL>
__global__ void __launch_bounds__(kSegThreads) segment_pass2(BatchArgs a, uint64_t n,
                                                             const uint32_t* __restrict__ skeys) {
  using M = Map<KIND, NC>;
  const int lane = threadIdx.x & 31;
  const uint64_t c = ((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5;
  const uint64_t nchunks = (n + 31) / 32;
  if (c >= nchunks) return;
  const uint8_t f = a.chunk_flags[c];
  if ((f & kNoHead) || !(f & kContOut)) return;
  const uint32_t d = a.dim, h = d / 2;
  const uint64_t end = min(c * 32 + 32, n);
  const uint32_t row = skeys[end - 1];
  double g[M::NE];
#pragma unroll
  for (int e = 0; e < M::NE; ++e)
    g[e] = M::ok(e, lane, d, h) ? a.part_last[c * d + M::idx(e, lane, h)] : 0.0;
  for (uint64_t c2 = c + 1; c2 < nchunks; ++c2) {
#pragma unroll
    for (int e = 0; e < M::NE; ++e)
      if (M::ok(e, lane, d, h)) g[e] += a.part_first[c2 * d + M::idx(e, lane, h)];
    const uint8_t f2 = a.chunk_flags[c2];
    if (!((f2 & kNoHead) && (f2 & kContOut))) break;
  }
  finish_row<KIND, NC, REL>(a, row, g, lane);
}

// ----------------------------------------------------------- dispatchers
template <int KIND, int NC>
void run_batch(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev) {
  auto rec = [&](int i) {
    if (ev && ev->enabled) LGD_CUDA(cudaEventRecord(ev->ev[i], st));
  };
  const uint32_t d = a.dim, k = a.k;
  const uint64_t P = a.P;
  const uint32_t dpad = (d + 3) & ~3u;
  const size_t smem = score_smem_bytes(d, k);
  const bool tma = (d % 4) == 0;
  rec(0);
  {
    const uint64_t blocks_needed = (P + kScoreWarps - 1) / kScoreWarps;
    int per_sm = 1;
    if (tma) {
      LGD_CUDA(cudaFuncSetAttribute(score_kernel<KIND, NC, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LGD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, score_kernel<KIND, NC, true>, kScoreWarps * 32, smem));
    } else {
      LGD_CUDA(cudaFuncSetAttribute(score_kernel<KIND, NC, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LGD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, score_kernel<KIND, NC, false>, kScoreWarps * 32, smem));
    }
    if (per_sm < 1) throw std::invalid_argument("batch shape exceeds shared memory (k, dim)");
    const uint64_t cap = (uint64_t)per_sm * a.sm_count;
    const unsigned grid = (unsigned)(blocks_needed < cap ? blocks_needed : cap);
    if (tma) {
      score_kernel<KIND, NC, true><<<grid, kScoreWarps * 32, smem, st>>>(a, dpad);
    } else {
      score_kernel<KIND, NC, false><<<grid, kScoreWarps * 32, smem, st>>>(a, dpad);
    }
    LGD_LAUNCH_CHECK();
  }
  loss_reduce_kernel<<<1, 1024, 0, st>>>(a.loss, P, a.batch_loss_out);
  LGD_LAUNCH_CHECK();
  rec(1);
  const uint64_t items = P * (k + 2);
  {
    size_t bytes = a.sort_temp_bytes;
    LGD_CUDA(cub::DeviceRadixSort::SortPairs(a.sort_temp, bytes, a.node_keys, a.skeys, a.iota,
                                             a.svals, (int64_t)items, 0, a.node_key_bits, st));
  }
  rec(2);
  {
    const unsigned grid = ceil_div(ceil_div(items, 32), kSegThreads / 32);
    segment_pass1<KIND, NC, false><<<grid, kSegThreads, 0, st>>>(a, items, a.skeys, a.svals);
    LGD_LAUNCH_CHECK();
    segment_pass2<KIND, NC, false><<<grid, kSegThreads, 0, st>>>(a, items, a.skeys);
    LGD_LAUNCH_CHECK();
  }
  rec(3);
  if (KIND != 0) {
    size_t bytes = a.sort_temp_bytes;
    LGD_CUDA(cub::DeviceRadixSort::SortPairs(a.sort_temp, bytes, a.rel_keys, a.skeys, a.iota,
                                             a.svals, (int64_t)P, 0, a.rel_key_bits, st));
    const unsigned grid = ceil_div(ceil_div(P, 32), kSegThreads / 32);
    segment_pass1<KIND, NC, true><<<grid, kSegThreads, 0, st>>>(a, P, a.skeys, a.svals);
    LGD_LAUNCH_CHECK();
    segment_pass2<KIND, NC, true><<<grid, kSegThreads, 0, st>>>(a, P, a.skeys);
    LGD_LAUNCH_CHECK();
  }
  rec(4);
}

template <int KIND>
void run_kind(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev) {
  const uint32_t lanes_elems = KIND == 2 ? a.dim / 2 : a.dim;
  const uint32_t nc = (lanes_elems + 31) / 32;
  if (nc <= 1) return run_batch<KIND, 1>(a, st, ev);
  if (nc <= 2) return run_batch<KIND, 2>(a, st, ev);
  if (nc <= 4) return run_batch<KIND, 4>(a, st, ev);
  if (nc <= 8) return run_batch<KIND, 8>(a, st, ev);
  throw std::invalid_argument("embedding dimension too large (max 256, ComplEx 512)");
}

}  // namespace

size_t batch_sort_temp_bytes(uint64_t max_items) {
  size_t bytes = 0;
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (int64_t)(max_items ? max_items : 1),
                                           0, 32));
  return bytes;
}

size_t score_smem_bytes(uint32_t dim, uint32_t k) {
  const size_t dpad = (dim + 3) & ~3u;
  const size_t warp_bytes = 2 * (size_t)(k + 3) * dpad * sizeof(float) + 2 * (size_t)k * 8;
  return 16 * kScoreWarps + kScoreWarps * warp_bytes;
}

void launch_train_batch(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev) {
  if (a.P == 0) return;
  switch (a.kind) {
    case 0:
      return run_kind<0>(a, st, ev);
    case 1:
      return run_kind<1>(a, st, ev);
    default:
      return run_kind<2>(a, st, ev);
  }
}

}  // namespace lgd
