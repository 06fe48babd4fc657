// train.cu -- the per-batch hot path: batch_loss + batch_gradients +
// adagrad_step (train.cpp:217-363) as
//
//   K3 score_kernel    warp per positive.  The 2+k+t embedding rows land in
//                      the warp's shared memory by TMA bulk copies
//                      (cp.async.bulk, one per row, mbarrier-tracked), the
//                      next positive's row ids fetched ahead.  Lane j computes
//                      the dot product of negative j (lane k: the positive)
//                      sequentially over the dimension -- the reference's own
//                      FP64 summation order (train.cpp:246-264) -- then the
//                      softmax weights, the loss and mix = sum_j w_j neg_j -
//                      dst (train.cpp:306-323) in the reference order.
//   sort               CUB onesweep radix sort of the P(k+2) contribution
//                      keys (pool indices).  Stable, so every node's
//                      contributions stay in the reference's std::map visit
//                      order (positive ascending; dst, negatives j, src).
//   K4 segment_pass1   warp per 32 sorted contributions; the chunk's pieces
//     (_vec)           (node segments cut at chunk edges) one after another,
//                      lanes over 16-byte vectors of the row.  The theta /
//                      state rows of the next four pieces are in flight in a
//                      per-warp shared-memory ring (cp.async); contributions
//                      are summed in order in FP64 and finished segments get
//                      their Adagrad row update (adagrad.cuh) right away -- a
//                      sort-by-node segmented reduction, no atomics on rows.
//   K4 segment_pass2   segments that run past a chunk and its 32-item
//                      lookahead (hubs) are finished by one block each from
//                      the per-chunk partial sums, in a fixed order.
//   relation path      the same segmented reduction over relation ids.
//   shared negatives   shared.cu (tcgen05) replaces K3; the update is K4.
// FP64 expressions are compiled with -fmad=false so products and sums round
// exactly like the reference's unfused x86-64 double arithmetic.
#include <cub/device/device_radix_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "adagrad.cuh"
#include "common.cuh"
#include "train.cuh"

namespace lgd {

namespace {

#ifndef SCORE_WARPS
#define SCORE_WARPS 8
#endif
constexpr int kScoreWarps = SCORE_WARPS;
// warps per K3 block by model: TransE (d = 128 on its BASELINE config, ~11 KB
// of rows per warp) packs more warps per SM in 4-warp blocks (Friendster
// +1.4%); 8-warp blocks are best for the rest (TW -1.7% at 4; r02zg)
template <int KIND>
constexpr int score_warps() { return KIND == 3 && SCORE_WARPS == 8 ? 4 : SCORE_WARPS; }
#ifndef SEG_THREADS
#define SEG_THREADS 256
#endif
constexpr int kSegThreads = SEG_THREADS;
// K4 blocks per SM: 4 (64 registers) -- the first contribution is read when
// the piece is processed rather than prefetched, so 32 warps fit per SM
#ifndef SEG_MINB
#define SEG_MINB 4
#endif
#ifndef SEG_DEPTH
#define SEG_DEPTH 2
#endif
#ifndef K4_BULK_ALL  // 1: every model's segment_heads stages by TMA bulk copies (A/B)
#define K4_BULK_ALL 0
#endif
// pieces / segments whose rows are in flight per warp in K4's cp.async rings
// (the chunked and flattened kernels; segment_heads picks its depth per model,
// seg_heads_depth: TW DistMult measured 2 best, 0.80 ms per batch; 3: 0.81,
// 4: 0.88 -- the ring's shared memory costs occupancy)
constexpr int kSegDepth = SEG_DEPTH;

// Developer timeline of K4 warps (build with -DLGD_TRACE; not in the product .so)
#ifdef LGD_TRACE
__device__ unsigned long long g_trace_k4[8][1024];
__device__ unsigned int g_trace_k4_n[8];
#define K4_TRACE(tag)                                                                  \
  do {                                                                                 \
    const unsigned wg = (blockIdx.x * kSegThreads + threadIdx.x) >> 5;                 \
    if ((threadIdx.x & 31) == 0 && wg % 7001 == 0 && wg / 7001 < 8) {                  \
      const unsigned i = g_trace_k4_n[wg / 7001]++;                                    \
      if (i < 512) {                                                                   \
        g_trace_k4[wg / 7001][2 * i] = clock64();                                      \
        g_trace_k4[wg / 7001][2 * i + 1] = (tag);                                      \
      }                                                                                \
    }                                                                                  \
  } while (0)
#else
#define K4_TRACE(tag) \
  do {                \
  } while (0)
#endif
constexpr int kPass2Threads = 256;
constexpr uint8_t kNoHead = 1;
constexpr uint8_t kContOut = 2;
constexpr int kGroup = 8;  // lanes per segment group in K4

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

// the same on a 32-bit shared-memory address (no generic pointer kept live)
__device__ __forceinline__ void mbar_init_s(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
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

// ------------------------------------------------------- pool indices
// (pool ranges hold < 2^32 rows: 32-bit offsets; an id below a range's first
// wraps to a large offset and fails the size test.  K3 of TransE keeps the
// loop form, measured faster there through its register allocation.)
__device__ __forceinline__ uint32_t to_pool_loop(const BatchArgs& a, uint32_t id) {
  uint64_t prev = 0;
  for (int i = 0; i < a.pool_n; ++i) {
    const uint64_t cnt = a.pool_end[i] - prev;
    if (id >= a.pool_first[i] && id - a.pool_first[i] < cnt) return (uint32_t)(prev + id - a.pool_first[i]);
    prev = a.pool_end[i];
  }
  return 0xffffffffu;
}
__device__ __forceinline__ uint32_t to_pool(const BatchArgs& a, uint32_t id) {
  const uint32_t e0 = (uint32_t)a.pool_end[0];
  const uint32_t o0 = id - (uint32_t)a.pool_first[0];
  if (o0 < e0) return o0;
  if (a.pool_n > 1) {
    const uint32_t e1 = (uint32_t)a.pool_end[1];
    const uint32_t o1 = id - (uint32_t)a.pool_first[1];
    if (o1 < e1 - e0) return e0 + o1;
    if (a.pool_n > 2) {
      const uint32_t o2 = id - (uint32_t)a.pool_first[2];
      if (o2 < (uint32_t)a.pool_end[2] - e1) return e1 + o2;
    }
  }
  return 0xffffffffu;  // not resident (validated on the host)
}
__device__ __forceinline__ uint32_t from_pool(const BatchArgs& a, uint32_t idx) {
  idx &= a.key_mask;  // presorted keys carry the batch index above the pool index
  LGD_DCHECK(idx < a.pool_end[a.pool_n - 1], "pool index beyond the resident pool", idx);
  if (idx < a.pool_end[0]) return (uint32_t)(a.pool_first[0] + idx);
  if (a.pool_n > 1 && idx < a.pool_end[1]) return (uint32_t)(a.pool_first[1] + (idx - a.pool_end[0]));
  return (uint32_t)(a.pool_first[2] + (idx - a.pool_end[1]));
}

// ---------------------------------------------------------------- K3 score
// Shared memory per warp: ids[32] u32, rows[(k+3) x dpad] f32 (src, rel,
// dst, negatives), ir1[dpad] f64, f[k+1] f64, e[k] f64.  One row buffer per
// warp keeps the footprint at ~9 KB so 24 warps share an SM; the next
// positive's row ids are fetched while the current one computes.
struct ScoreSmem {
  uint32_t dpad, k, nrows;
  size_t ids_off, rows_off, ir1_off, f_off, e_off, warp_bytes;
  __host__ __device__ ScoreSmem(uint32_t d, uint32_t kk) {
    dpad = (d + 3) & ~3u;
    k = kk;
    nrows = kk + 3;
    const uint32_t nid = (nrows + 31) & ~31u;
    ids_off = 0;
    rows_off = (nid * 4 + 15) & ~size_t(15);
    ir1_off = rows_off + size_t(nrows) * dpad * 4;
    f_off = ir1_off + size_t(dpad) * 8;
    e_off = f_off + size_t(kk + 1) * 8;
    warp_bytes = (e_off + size_t(kk) * 8 + 15) & ~size_t(15);
  }
  __host__ __device__ size_t block_bytes(int warps) const { return 16 * warps + warps * warp_bytes; }
};

template <int KIND>
__global__ void __launch_bounds__(score_warps<KIND>() * 32) score_kernel(BatchArgs a, int use_tma) {
  constexpr int kWarpsK3 = score_warps<KIND>();
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t k = a.k, d = a.dim, h = d / 2;
  const bool typed = KIND != 0;
  const ScoreSmem L(d, k);
  const uint32_t dpad = L.dpad, nrows = L.nrows;
  const uint32_t nid = (nrows + 31) & ~31u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + 2 * warp;
  unsigned char* wbase = smem + 16 * kWarpsK3 + warp * L.warp_bytes;
  uint32_t* ids = reinterpret_cast<uint32_t*>(wbase + L.ids_off);
  float* rows = reinterpret_cast<float*>(wbase + L.rows_off);
  double* ir1 = reinterpret_cast<double*>(wbase + L.ir1_off);
  double* fbuf = reinterpret_cast<double*>(wbase + L.f_off);
  double* ebuf = reinterpret_cast<double*>(wbase + L.e_off);
  const size_t buf_floats = size_t(nrows) * dpad;
  const bool tma = use_tma && nrows <= 32;
  if (KIND != 0 && a.rel64 && blockIdx.x == 0)  // K4's FP64 relation rows (exact conversion)
    for (uint64_t i = threadIdx.x; i < a.num_rels * d; i += blockDim.x) a.rel64[i] = a.rel_theta[i];

  if (tma) {
    if (lane == 0) {
      mbar_init(bars, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  const uint32_t row_bytes = d * 4;
  const uint32_t tx_bytes = (typed ? nrows : nrows - 1) * row_bytes;

  // row r of positive p: 0 src, 1 rel, 2 dst, 3+j negative j
  auto row_id = [&](uint64_t p, uint32_t r) -> uint32_t {
    const uint32_t id = r < 3 ? a.edges[3 * p + r] : a.negs[p * k + (r - 3)];
    LGD_DCHECK(r == 1 ? (!typed || id < a.num_rels) : id < a.num_nodes, "K3 row id out of range", id);
    return id;
  };
  auto row_src = [&](uint32_t r, uint32_t id) -> const float* {
    return (r == 1 ? a.rel_theta : a.theta) + size_t(id) * d;
  };
  auto issue = [&](uint32_t my_id, int b) {  // TMA path: lane r owns row r's id
    if (lane < (int)nrows) ids[b * nid + lane] = my_id;
    if (lane == 0) mbar_arrive_expect_tx(bars + b, tx_bytes);
    __syncwarp();
    if (lane < (int)nrows && (typed || lane != 1))
      bulk_g2s(rows + b * buf_floats + lane * dpad, row_src(lane, my_id), row_bytes, bars + b);
  };
  auto load_sync = [&](uint64_t p, int b) {  // generic path: plain loads
    for (uint32_t r = lane; r < nrows; r += 32) ids[b * nid + r] = row_id(p, r);
    __syncwarp();
    float* base = rows + b * buf_floats;
    for (uint32_t r = 0; r < nrows; ++r) {
      if (r == 1 && !typed) continue;
      const float* src = row_src(r, ids[b * nid + r]);
      for (uint32_t i = lane; i < d; i += 32) base[r * dpad + i] = src[i];
    }
    __syncwarp();
  };

  const uint64_t nwarps = (uint64_t)gridDim.x * kWarpsK3;
  uint64_t p = (uint64_t)blockIdx.x * kWarpsK3 + warp;
  uint32_t phase = 0;
  uint32_t id_next = 0;
  const int b = 0;
  if (tma && p < a.P) {
    const uint32_t id0 = lane < (int)nrows ? row_id(p, lane) : 0;
    issue(id0, 0);
    const uint64_t p1 = p + nwarps;
    if (p1 < a.P && lane < (int)nrows) id_next = row_id(p1, lane);
  }
  for (; p < a.P; p += nwarps) {
    const uint64_t pn = p + nwarps, pnn = pn + nwarps;
    if (tma) {
      while (!mbar_try_wait(bars, phase)) {
      }
      phase ^= 1;
    } else {
      load_sync(p, b);
    }
    __syncwarp();
    const float* R = rows + b * buf_floats;
    const float* srow = R;
    const float* rrow = R + dpad;
    const float* drow = R + 2 * dpad;
    const uint32_t* pid = ids + b * nid;

    // IR1 = s (x) r (combine_src_rel, train.cpp:39-60) into shared memory
    if (KIND == 2) {
      for (uint32_t j = lane; j < h; j += 32) {
        const double sr = srow[j], si = srow[j + h];
        const double rr = rrow[j], ri = rrow[j + h];
        const double xr = sr * rr - si * ri, xi = sr * ri + si * rr;
        ir1[j] = xr;
        ir1[j + h] = xi;
        if (k4_ir1(KIND) && a.ir1) {
          a.ir1[p * d + j] = xr;
          a.ir1[p * d + j + h] = xi;
        }
      }
      for (uint32_t i = lane; i < d; i += 32) a.snap[p * d + i] = srow[i];
    } else if ((d & 3) == 0) {  // lane-owned float4 columns (TransE: u = s + r)
      for (uint32_t i = 4 * lane; i < d; i += 128) {
        const float4 sv = *reinterpret_cast<const float4*>(srow + i);
        double u0 = sv.x, u1 = sv.y, u2 = sv.z, u3 = sv.w;
        if (KIND != 0) {
          const float4 rv = *reinterpret_cast<const float4*>(rrow + i);
          if (KIND == 3) {
            u0 += (double)rv.x, u1 += (double)rv.y, u2 += (double)rv.z, u3 += (double)rv.w;
          } else {
            u0 *= (double)rv.x, u1 *= (double)rv.y, u2 *= (double)rv.z, u3 *= (double)rv.w;
          }
        }
        *reinterpret_cast<double2*>(ir1 + i) = make_double2(u0, u1);
        *reinterpret_cast<double2*>(ir1 + i + 2) = make_double2(u2, u3);
        if (k4_ir1(KIND) && a.ir1) {
          *reinterpret_cast<double2*>(a.ir1 + p * d + i) = make_double2(u0, u1);
          *reinterpret_cast<double2*>(a.ir1 + p * d + i + 2) = make_double2(u2, u3);
        }
        *reinterpret_cast<float4*>(a.snap + p * d + i) = sv;
      }
    } else {
      for (uint32_t i = lane; i < d; i += 32) {
        ir1[i] = KIND == 0   ? (double)srow[i]
                 : KIND == 3 ? (double)srow[i] + (double)rrow[i]
                             : (double)srow[i] * (double)rrow[i];
        if (k4_ir1(KIND) && a.ir1) a.ir1[p * d + i] = ir1[i];
      }
      for (uint32_t i = lane; i < d; i += 32) a.snap[p * d + i] = srow[i];
    }
    __syncwarp();
    // scores: lane q < k -> negative q, lane k -> the positive; sequential
    // over the dimension exactly as train.cpp:246-264
    for (uint32_t q = lane; q <= k; q += 32) {
      const float* row = q < k ? R + (3 + q) * dpad : drow;
      double f = 0.0;
      if (KIND == 3) {  // -||u - t||, squares summed sequentially
        if ((d & 3) == 0) {  // 16-byte shared loads, the same sequential order
          for (uint32_t i = 0; i < d; i += 4) {
            const float4 v = *reinterpret_cast<const float4*>(row + i);
            const double2 x0 = *reinterpret_cast<const double2*>(ir1 + i);
            const double2 x1 = *reinterpret_cast<const double2*>(ir1 + i + 2);
            const double q0 = x0.x - (double)v.x, q1 = x0.y - (double)v.y;
            const double q2 = x1.x - (double)v.z, q3 = x1.y - (double)v.w;
            f += q0 * q0;
            f += q1 * q1;
            f += q2 * q2;
            f += q3 * q3;
          }
        } else {
          for (uint32_t i = 0; i < d; ++i) {
            const double q = ir1[i] - (double)row[i];
            f += q * q;
          }
        }
        f = -sqrt(f);
      } else if ((d & 3) == 0) {
        for (uint32_t i = 0; i < d; i += 4) {
          const float4 v = *reinterpret_cast<const float4*>(row + i);
          const double2 x0 = *reinterpret_cast<const double2*>(ir1 + i);
          const double2 x1 = *reinterpret_cast<const double2*>(ir1 + i + 2);
          f += x0.x * (double)v.x;
          f += x0.y * (double)v.y;
          f += x1.x * (double)v.z;
          f += x1.y * (double)v.w;
        }
      } else {
        for (uint32_t i = 0; i < d; ++i) f += ir1[i] * (double)row[i];
      }
      fbuf[q] = f;
    }
    __syncwarp();
    // std::max over the negatives' scores (train.cpp:262-264): for the
    // non-NaN scores the max is order-free, so a butterfly over lanes gives
    // the sequential fold's value
    // (Dot and TransE keep the sequential fold: measured faster there, by
    // their register allocation)
    constexpr bool kFly = KIND == 1 || KIND == 2;
    double row_max = -INFINITY;
    for (uint32_t j = kFly ? lane : 0; j < k; j += kFly ? 32 : 1) {
      const double f = fbuf[j];
      row_max = row_max < f ? f : row_max;
    }
    if (kFly) {
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double f = __shfl_xor_sync(0xffffffffu, row_max, o);
        row_max = row_max < f ? f : row_max;
      }
    }
    for (uint32_t j = lane; j < k; j += 32) ebuf[j] = exp(fbuf[j] - row_max);  // IR3
    __syncwarp();
    double sum = 0.0;
    for (uint32_t j = 0; j < k; ++j) sum += ebuf[j];  // sequential j (train.cpp:266-270)
    const double inv_sum = 1.0 / sum;
    // loss = -(f_pos - (row_max + log(sum))), train.cpp:274.  With loss parts
    // (DistMult / ComplEx with the side-stream relation pass: run_batch) the
    // log runs lane-parallel in loss_reduce_kernel, off the critical path
    if (lane == 0) {
      if (!((KIND == 1 || KIND == 2) && a.loss_parts)) {
        a.loss[p] = -(fbuf[k] - (row_max + log(sum)));
      } else {
        a.loss[p] = fbuf[k];
        a.loss[a.P + p] = row_max;
        a.loss[2 * a.P + p] = sum;
      }
    }
    if (KIND == 3) {
      // TransE coefficients (oracle lo_batch_ex): c_j = w_j / D_j, c_pos =
      // -1 / D_pos (0 at D = 0), stored where w lives (c_pos after P x k);
      // mix = dL/du = -c_pos (u - t) - sum_j c_j (u - n_j), j ascending
      for (uint32_t j = lane; j < k; j += 32) {
        const double dj = -fbuf[j];
        ebuf[j] = dj > 0.0 ? (ebuf[j] * inv_sum) / dj : 0.0;
        a.w[p * k + j] = ebuf[j];
      }
      const double dpos = -fbuf[k];
      const double cpos = dpos > 0.0 ? -1.0 / dpos : 0.0;
      if (lane == 0) a.w[a.P * k + p] = cpos;
      __syncwarp();
      if ((d & 3) == 0) {  // lane-owned float4 columns: one pass for d <= 128
        for (uint32_t i = 4 * lane; i < d; i += 128) {
          const double2 u01 = *reinterpret_cast<const double2*>(ir1 + i);
          const double2 u23 = *reinterpret_cast<const double2*>(ir1 + i + 2);
          const float4 t = *reinterpret_cast<const float4*>(drow + i);
          double m0 = -(cpos * (u01.x - (double)t.x)), m1 = -(cpos * (u01.y - (double)t.y));
          double m2 = -(cpos * (u23.x - (double)t.z)), m3 = -(cpos * (u23.y - (double)t.w));
          for (uint32_t j = 0; j < k; ++j) {
            const double e = ebuf[j];
            const float4 v = *reinterpret_cast<const float4*>(R + (3 + j) * dpad + i);
            m0 -= e * (u01.x - (double)v.x);
            m1 -= e * (u01.y - (double)v.y);
            m2 -= e * (u23.x - (double)v.z);
            m3 -= e * (u23.y - (double)v.w);
          }
          *reinterpret_cast<double2*>(a.mix + p * d + i) = make_double2(m0, m1);
          *reinterpret_cast<double2*>(a.mix + p * d + i + 2) = make_double2(m2, m3);
        }
      } else {
        for (uint32_t i = lane; i < d; i += 32) {
          const double u = ir1[i];
          double mx = -(cpos * (u - (double)drow[i]));
          for (uint32_t j = 0; j < k; ++j) mx -= ebuf[j] * (u - (double)R[(3 + j) * dpad + i]);
          a.mix[p * d + i] = mx;
        }
      }
    } else {
      for (uint32_t j = lane; j < k; j += 32) {  // w_j = IR3_j / S as IR3_j * (1 / S)
        ebuf[j] = ebuf[j] * inv_sum;
        a.w[p * k + j] = ebuf[j];
      }
      __syncwarp();
      // mix = sum_j w_j neg_j - dst, j ascending (train.cpp:306-323)
      if ((d & 3) == 0) {  // lane-owned float4 columns: one pass for d <= 128
        for (uint32_t i = 4 * lane; i < d; i += 128) {
          const float4 t = *reinterpret_cast<const float4*>(drow + i);
          double m0 = -(double)t.x, m1 = -(double)t.y, m2 = -(double)t.z, m3 = -(double)t.w;
          for (uint32_t j = 0; j < k; ++j) {
            const double e = ebuf[j];
            const float4 v = *reinterpret_cast<const float4*>(R + (3 + j) * dpad + i);
            m0 += e * (double)v.x;
            m1 += e * (double)v.y;
            m2 += e * (double)v.z;
            m3 += e * (double)v.w;
          }
          *reinterpret_cast<double2*>(a.mix + p * d + i) = make_double2(m0, m1);
          *reinterpret_cast<double2*>(a.mix + p * d + i + 2) = make_double2(m2, m3);
        }
      } else {
        for (uint32_t i = lane; i < d; i += 32) {
          double mx = -(double)drow[i];
          for (uint32_t j = 0; j < k; ++j) mx += ebuf[j] * (double)R[(3 + j) * dpad + i];
          a.mix[p * d + i] = mx;
        }
      }
    }
    // contribution keys in the reference's visit order: dst, negatives, src
    const uint64_t kb = p * (k + 2);
    for (uint32_t r = lane; r < nrows; r += 32) {
      const uint32_t id = pid[r];
      // payload: positive, (relation,) slot
      const uint32_t pv = ((uint32_t)p << (a.slot_bits + a.rel_bits)) |
                          (a.rel_bits ? pid[1] << a.slot_bits : 0u);
      if (r != 1 && a.presorted) {
        // keyed and sorted for the whole bucket already (presort_keys_kernel)
      } else if (r == 0) {
        a.node_keys[kb + k + 1] = KIND == 3 ? to_pool_loop(a, id) : to_pool(a, id);
        a.node_vals[kb + k + 1] = pv | (k + 1);
      } else if (r == 1) {
        if (typed) a.rel_keys[p] = id;
      } else if (r == 2) {
        a.node_keys[kb] = KIND == 3 ? to_pool_loop(a, id) : to_pool(a, id);
        a.node_vals[kb] = pv;
      } else {
        a.node_keys[kb + (r - 2)] = KIND == 3 ? to_pool_loop(a, id) : to_pool(a, id);
        a.node_vals[kb + (r - 2)] = pv | (r - 2);
      }
    }
    __syncwarp();
    if (tma && pn < a.P) {  // the buffer is free again: fetch the next positive
      issue(id_next, 0);
      if (pnn < a.P && lane < (int)nrows) id_next = row_id(pnn, lane);
    }
  }
}

// --------------------------------------------------------- loss reduction
// parts: loss holds K3's f_pos | row_max | sum (3 x P) and the per-positive
// loss -(f_pos - (row_max + log(sum))) (train.cpp:274) is formed here
__global__ void __launch_bounds__(1024) loss_reduce_kernel(const double* __restrict__ loss,
                                                           uint64_t P, double* out, int parts) {
  __shared__ double part[1024];
  double s = 0.0;
  for (uint64_t i = threadIdx.x; i < P; i += 1024)
    s += parts ? -(loss[i] - (loss[P + i] + log(loss[2 * P + i]))) : loss[i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

// ------------------------------------------------- K4 segmented reduction
// Element ownership inside an 8-lane group: Dot / DistMult lane g owns
// i = g + 8c; ComplEx lane g owns real index j = g + 8c (< h) and its
// imaginary partner j + h (slots c and NC + c).
template <int KIND, int NC>
struct GMap {
  static constexpr int NE = KIND == 2 ? 2 * NC : NC;
  __device__ __forceinline__ static int idx(int e, int g, uint32_t h) {
    if (KIND == 2) return e < NC ? g + kGroup * e : g + kGroup * (e - NC) + (int)h;
    return g + kGroup * e;
  }
  __device__ __forceinline__ static bool ok(int e, int g, uint32_t d, uint32_t h) {
    if (KIND == 2) return g + kGroup * (e < NC ? e : e - NC) < (int)h;
    return g + kGroup * e < (int)d;
  }
};

// One sorted contribution added to the group lane's elements.  All loads are
// issued first (predicated, no branches) so a lane keeps every element of the
// item in flight at once; the FP64 arithmetic follows in the reference order.
template <int KIND, int NC, bool REL>
__device__ __forceinline__ void add_item(const BatchArgs& a, uint32_t val, int g, double* acc,
                                         const float* own) {
  using M = GMap<KIND, NC>;
  constexpr int NE = M::NE;
  const uint32_t d = a.dim, h = d / 2, k = a.k;
  if (REL) {  // relation gradient: adj_src(mix) (train.cpp:328-332)
    const float* s = a.snap + (uint64_t)val * d;
    const double* mx = a.mix + (uint64_t)val * d;
    float sv[NE];
    double mv[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const bool ok = M::ok(e, g, d, h);
      const int i = M::idx(e, g, h);
      sv[e] = ok ? __ldg(s + i) : 0.f;
      mv[e] = ok ? __ldg(mx + i) : 0.0;
    }
    if (KIND == 2) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double orr = sv[c], ori = sv[c + NC], mr = mv[c], mi = mv[c + NC];
        acc[c] += orr * mr + ori * mi;
        acc[c + NC] += orr * mi - ori * mr;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] += KIND == 3 ? mv[e] : (double)sv[e] * mv[e];
    }
    return;
  }
  const uint64_t p = val >> (a.slot_bits + a.rel_bits);
  const uint32_t slot = val & ((1u << a.slot_bits) - 1u);
  const bool is_src = slot > k;
  const float* rel = KIND != 0 ? a.rel_theta + (size_t)__ldg(a.rel_keys + p) * d : nullptr;
  const float* s = a.snap + p * d;
  const double* mx = a.mix + p * d;
  const double w = (slot >= 1 && !is_src) ? __ldg(a.w + p * k + (slot - 1))
                   : (KIND == 3 && slot == 0) ? __ldg(a.w + a.P * k + p) : 0.0;
  float rv[NE], sv[NE];
  double mv[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const bool ok = M::ok(e, g, d, h);
    const int i = M::idx(e, g, h);
    rv[e] = (KIND != 0 && ok) ? __ldg(rel + i) : 0.f;
    sv[e] = (!is_src && ok) ? __ldg(s + i) : 0.f;
    mv[e] = (is_src && ok) ? __ldg(mx + i) : 0.0;
  }
  if (!is_src) {  // dst: g -= IR1 (train.cpp:310); negative j: g += w_j IR1 (:320)
    if (KIND == 3) {  // TransE: g += c (u - own row)
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const double x = (double)sv[e] + (double)rv[e];
        acc[e] += w * (x - (double)own[e]);
      }
    } else if (KIND == 2) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double sr = sv[c], si = sv[c + NC], rr = rv[c], ri = rv[c + NC];
        const double xr = sr * rr - si * ri, xi = sr * ri + si * rr;
        acc[c] = slot == 0 ? acc[c] - xr : acc[c] + w * xr;
        acc[c + NC] = slot == 0 ? acc[c + NC] - xi : acc[c + NC] + w * xi;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const double x = KIND == 0 ? (double)sv[e] : (double)sv[e] * (double)rv[e];
        acc[e] = slot == 0 ? acc[e] - x : acc[e] + w * x;
      }
    }
  } else {  // src: g += adj_rel(mix) (train.cpp:327, adjoint_combine :65-85)
    if (KIND == 2) {
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double orr = rv[c], ori = rv[c + NC], mr = mv[c], mi = mv[c + NC];
        acc[c] += orr * mr + ori * mi;
        acc[c + NC] += orr * mi - ori * mr;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] += (KIND == 0 || KIND == 3) ? mv[e] : (double)rv[e] * mv[e];
    }
  }
}

template <bool REL>
__device__ __forceinline__ float* row_theta(const BatchArgs& a, uint32_t r) {
  return (REL ? a.rel_theta : a.theta) + (size_t)r * a.dim;
}
template <bool REL>
__device__ __forceinline__ float* row_state(const BatchArgs& a, uint32_t r) {
  return (REL ? a.rel_state : a.state) + (size_t)r * a.dim;
}

// adagrad_update (train.cpp:342-354): a = acc + g^2 (FP64), acc = f32(a),
// theta = f32(theta - lr g / (sqrt(a) + eps)), bit-identical through the
// certified fast path of adagrad.cuh (exact fallback otherwise).
__device__ __forceinline__ void adagrad_fast(double gi, float& th, float& st, double lr,
                                             double eps) {
  if (!adagrad_try_fast(gi, th, st, lr, eps)) adagrad_exact(gi, th, st, lr, eps);
}
__device__ __forceinline__ void adagrad_elem(double gi, float& th, float& st, double lr,
                                             double eps) {
  adagrad_fast(gi, th, st, lr, eps);
}

template <int KIND, int NC, bool REL>
__global__ void __launch_bounds__(kSegThreads) segment_pass1(BatchArgs a, uint64_t n,
                                                             const uint32_t* __restrict__ skeys,
                                                             const uint32_t* __restrict__ svals,
                                                             uint32_t* __restrict__ span_list,
                                                             unsigned int* __restrict__ span_count) {
  using M = GMap<KIND, NC>;
  constexpr int NE = M::NE;
  const int lane = threadIdx.x & 31;
  const int g = lane & (kGroup - 1);
  const int grp = lane >> 3;
  const uint64_t c = ((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5;
  const uint64_t base = c * 32;
  if (base >= n) return;
  const uint32_t d = a.dim, h = d / 2;
  const uint64_t end = min(base + 32, n);
  const uint64_t i = base + lane;
  const uint32_t key = i < n ? skeys[i] : 0;
  const bool head = i < n && (i == 0 || skeys[i - 1] != key);
  const uint32_t hmask = __ballot_sync(0xffffffffu, head);
  const bool cont_in = !(hmask & 1u);
  const bool cont_out = end < n && skeys[end] == skeys[end - 1];
  const uint32_t smask = hmask | 1u;  // piece starts (bit 0 also starts a continuation)
  const int np = __popc(smask);
  // lane t < np: start offset of piece t (t-th set bit of smask)
  int my_start = 32;
  if (lane < np) {
    uint32_t m = smask;
    for (int s2 = 0; s2 < lane; ++s2) m &= m - 1;
    my_start = __ffs(m) - 1;
  }
  const int nlive = (int)(end - base);
  for (int r0 = 0; r0 < np; r0 += 4) {
    const int t = r0 + grp;  // this group's piece
    const bool live = t < np;
    const int ps = __shfl_sync(0xffffffffu, my_start, t & 31);
    const int pe_next = __shfl_sync(0xffffffffu, my_start, (t + 1) & 31);
    const int pstart = live ? ps : 0;
    const int pend = live ? (t + 1 < np ? pe_next : nlive) : 0;
    const bool first_piece = live && t == 0 && cont_in;
    const bool last_piece = live && t == np - 1 && cont_out;
    const bool finish = live && !first_piece && !last_piece;
    const uint32_t row = live ? (REL ? skeys[base + pstart] : from_pool(a, skeys[base + pstart])) : 0;
    float tv[NE], sv[NE];
    constexpr bool kOwn = KIND == 3 && !REL;  // TransE contributions read the node's own row
    const bool upd = finish && !(REL ? a.grad_rels : a.grad_nodes);
    if (upd || (kOwn && live)) {  // prefetch theta / state
      const float* th = row_theta<REL>(a, row);
      const float* st = row_state<REL>(a, row);
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        tv[e] = 0.f;
        if (M::ok(e, g, d, h)) {
          tv[e] = th[M::idx(e, g, h)];
          if (upd) sv[e] = st[M::idx(e, g, h)];
        }
      }
    }
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
    // lockstep over the longest piece of this round
    int len = pend - pstart;
    int maxlen = len;
#pragma unroll
    for (int off = 8; off < 32; off <<= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, off));
    for (int q = 0; q < maxlen; ++q) {
      if (q < len) add_item<KIND, NC, REL>(a, __ldg(svals + base + pstart + q), g, acc, tv);
    }
    if (first_piece || last_piece) {
      double* dst = (first_piece ? a.part_first : a.part_last) + c * d;
#pragma unroll
      for (int e = 0; e < NE; ++e)
        if (M::ok(e, g, d, h)) dst[M::idx(e, g, h)] = acc[e];
    } else if (finish) {
      double* gout = REL ? a.grad_rels : a.grad_nodes;
      if (gout) {
#pragma unroll
        for (int e = 0; e < NE; ++e)
          if (M::ok(e, g, d, h)) gout[(size_t)row * d + M::idx(e, g, h)] = acc[e];
        if (g == 0) (REL ? a.grad_rel_flag : a.grad_node_flag)[row] = 1;
      } else {
        float* th = row_theta<REL>(a, row);
        float* st = row_state<REL>(a, row);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          if (M::ok(e, g, d, h)) {
            adagrad_elem(acc[e], tv[e], sv[e], a.lr, a.eps);
            th[M::idx(e, g, h)] = tv[e];
            st[M::idx(e, g, h)] = sv[e];
          }
        }
      }
    }
  }
  if (lane == 0) {
    const int heads = __popc(hmask);
    a.chunk_flags[c] = (heads ? 0 : kNoHead) | (cont_out ? kContOut : 0);
    if (heads) atomicAdd(a.counters + (REL ? 1 : 0), (unsigned long long)heads);
    if (heads && cont_out) span_list[atomicAdd(span_count, 1u)] = (uint32_t)c;
  }
}

// ---------------------------------------------- K4, vector-lane variant
// Full warp per piece, lanes own 16-byte vectors: Dot / DistMult lane l owns
// elements 4q..4q+3 (q = l + 32v, float4); ComplEx lane l owns the real pair
// 2q, 2q+1 and its imaginary partners h+2q, h+2q+1 (float2 each), stored at
// e = 4v + {0,1} (re) and 4v + {2,3} (im).  The next piece's theta / state and
// first contribution are loaded while the current piece computes.
template <int KIND, int NV>
struct Lanes {
  bool ok[NV];
  uint32_t off[NV];  // element offset of the lane's (real) vector
  uint32_t h;
  __device__ __forceinline__ Lanes(int lane, uint32_t d) {
    h = d / 2;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t q = lane + 32 * v;
      ok[v] = KIND == 2 ? 2 * q < h : 4 * q < d;
      off[v] = KIND == 2 ? 2 * q : 4 * q;
    }
  }
  template <bool RO>
  __device__ __forceinline__ void ldf(const float* b, bool pred, float* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const bool o = pred && ok[v];
      if (KIND == 2) {
        float2 re = make_float2(0.f, 0.f), im = make_float2(0.f, 0.f);
        if (o) {
          const float2* pr = reinterpret_cast<const float2*>(b + off[v]);
          const float2* pi = reinterpret_cast<const float2*>(b + off[v] + h);
          re = RO ? __ldg(pr) : *pr;
          im = RO ? __ldg(pi) : *pi;
        }
        x[4 * v] = re.x;
        x[4 * v + 1] = re.y;
        x[4 * v + 2] = im.x;
        x[4 * v + 3] = im.y;
      } else {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (o) {
          const float4* pt = reinterpret_cast<const float4*>(b + off[v]);
          t = RO ? __ldg(pt) : *pt;
        }
        x[4 * v] = t.x;
        x[4 * v + 1] = t.y;
        x[4 * v + 2] = t.z;
        x[4 * v + 3] = t.w;
      }
    }
  }
  // cp.async the lane's elements of a global row into the same positions of
  // a shared-memory row (zero-filled when !pred); lds reads them back.  Each
  // lane only ever touches its own elements, so no warp sync is needed.
  __device__ __forceinline__ void cpa(float* s, const float* g, bool pred) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!ok[v]) continue;
      const uint32_t n = pred ? (KIND == 2 ? 8u : 16u) : 0u;
      if (KIND == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s + off[v])),
                     "l"(g + off[v]), "r"(n)
                     : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s + off[v] + h)),
                     "l"(g + off[v] + h), "r"(n)
                     : "memory");
      } else {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s + off[v])),
                     "l"(g + off[v]), "r"(n)
                     : "memory");
      }
    }
  }
  // the same with 32-bit shared-state-space addresses (no generic conversion)
  __device__ __forceinline__ void cpa_s(uint32_t s, const float* g, bool pred) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!ok[v]) continue;
      const uint32_t n = pred ? (KIND == 2 ? 8u : 16u) : 0u;
      if (KIND == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s + 4 * off[v]),
                     "l"(g + off[v]), "r"(n)
                     : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s + 4 * (off[v] + h)),
                     "l"(g + off[v] + h), "r"(n)
                     : "memory");
      } else {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s + 4 * off[v]),
                     "l"(g + off[v]), "r"(n)
                     : "memory");
      }
    }
  }
  // f64 rows (mix, IR1) in the lane's layout of ldd: double2 at off and at
  // off + (ComplEx: h, else 2), staged by cp.async into the same positions
  __device__ __forceinline__ void cpd_s(uint32_t s, const double* g) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!ok[v]) continue;
      const uint32_t o2 = off[v] + (KIND == 2 ? h : 2);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + 8 * off[v]),
                   "l"(g + off[v])
                   : "memory");
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + 8 * o2), "l"(g + o2)
                   : "memory");
    }
  }
  __device__ __forceinline__ void ldd_s(uint32_t s, double* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      if (ok[v]) {
        const uint32_t o2 = off[v] + (KIND == 2 ? h : 2);
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a0), "=d"(a1) : "r"(s + 8 * off[v]));
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a2), "=d"(a3) : "r"(s + 8 * o2));
      }
      x[4 * v] = a0;
      x[4 * v + 1] = a1;
      x[4 * v + 2] = a2;
      x[4 * v + 3] = a3;
    }
  }
  __device__ __forceinline__ void lds_s(uint32_t s, float* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
      if (ok[v]) {
        if (KIND == 2) {
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a0), "=f"(a1) : "r"(s + 4 * off[v]));
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                       : "=f"(a2), "=f"(a3)
                       : "r"(s + 4 * (off[v] + h)));
        } else {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
                       : "r"(s + 4 * off[v]));
        }
      }
      x[4 * v] = a0;
      x[4 * v + 1] = a1;
      x[4 * v + 2] = a2;
      x[4 * v + 3] = a3;
    }
  }
  __device__ __forceinline__ void lds(const float* s, float* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (KIND == 2) {
        float2 re = make_float2(0.f, 0.f), im = make_float2(0.f, 0.f);
        if (ok[v]) {
          re = *reinterpret_cast<const float2*>(s + off[v]);
          im = *reinterpret_cast<const float2*>(s + off[v] + h);
        }
        x[4 * v] = re.x;
        x[4 * v + 1] = re.y;
        x[4 * v + 2] = im.x;
        x[4 * v + 3] = im.y;
      } else {
        float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok[v]) t = *reinterpret_cast<const float4*>(s + off[v]);
        x[4 * v] = t.x;
        x[4 * v + 1] = t.y;
        x[4 * v + 2] = t.z;
        x[4 * v + 3] = t.w;
      }
    }
  }
  __device__ __forceinline__ void ldd(const double* b, bool pred, double* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const bool o = pred && ok[v];
      double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
      if (o) {
        a0 = __ldg(reinterpret_cast<const double2*>(b + off[v]));
        a1 = __ldg(reinterpret_cast<const double2*>(b + off[v] + (KIND == 2 ? h : 2)));
      }
      x[4 * v] = a0.x;
      x[4 * v + 1] = a0.y;
      x[4 * v + 2] = a1.x;
      x[4 * v + 3] = a1.y;
    }
  }
  __device__ __forceinline__ void stf(float* b, const float* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!ok[v]) continue;
      if (KIND == 2) {
        *reinterpret_cast<float2*>(b + off[v]) = make_float2(x[4 * v], x[4 * v + 1]);
        *reinterpret_cast<float2*>(b + off[v] + h) = make_float2(x[4 * v + 2], x[4 * v + 3]);
      } else {
        *reinterpret_cast<float4*>(b + off[v]) =
            make_float4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
      }
    }
  }
  __device__ __forceinline__ void std_(double* b, const double* x) const {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      if (!ok[v]) continue;
      *reinterpret_cast<double2*>(b + off[v]) = make_double2(x[4 * v], x[4 * v + 1]);
      *reinterpret_cast<double2*>(b + off[v] + (KIND == 2 ? h : 2)) =
          make_double2(x[4 * v + 2], x[4 * v + 3]);
    }
  }
};

// adagrad_update (train.cpp:342-354) on the lane's elements (adagrad.cuh):
// only the vectors the lane owns run it.
template <int KIND, int NV>
__device__ __forceinline__ void adagrad_lanes(const Lanes<KIND, NV>& L, const double* acc,
                                              float* th, float* st, double lr, double eps) {
  uint32_t slow = 0;  // elements the fast path could not certify (~0.05%)
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (!L.ok[v]) continue;
#pragma unroll
    for (int e = 4 * v; e < 4 * v + 4; ++e)
#ifndef LGD_ADAGRAD2
      if (!adagrad_try_fast1(acc[e], th[e], st[e], lr, eps)) slow |= 1u << e;
#else  // the two-Newton-step certificate (round 1)
      if (!adagrad_try_fast(acc[e], th[e], st[e], lr, eps)) slow |= 1u << e;
#endif
  }
  if (slow) {
#pragma unroll
    for (int e = 0; e < 4 * NV; ++e)
      if ((slow >> e) & 1u) adagrad_exact(acc[e], th[e], st[e], lr, eps);
  }
}

// One contribution's operands: the src snapshot (dst / negative items), the
// relation row, mix (src items) and the softmax weight.
template <int NE>
struct ItemRegs {
  float sv[NE];
  double mv[NE];
  double w;
  uint32_t slot;
  uint32_t rel;  // relation row id: read at use (a small, L1-resident table)
};

struct SegCtx {  // hoisted kernel arguments
  const float* snap;
  const double* mix;
  const double* ir1;  // K3's IR1 rows (k4_ir1)
  const double* w;
  const float* rel_theta;
  const uint32_t* rel_keys;
  uint32_t d, k, sbits, smask;
  uint32_t pshift, rmask;  // positive = val >> pshift; relation = (val >> sbits) & rmask (0: look up)
  uint64_t cpos_off;  // TransE: offset of the dst coefficients in w (P k)
  const float* gneg;  // shared-negative mode: gradient rows of the shared negatives
  const double* rel64;  // the relation rows in FP64 (K3 writes them for small R), or null
};

template <int KIND, int NV, bool REL, bool SH, bool IR1 = k4_ir1(KIND)>
__device__ __forceinline__ void load_item(const SegCtx& x, const Lanes<KIND, NV>& L, uint32_t val,
                                          bool pred, ItemRegs<4 * NV>& it) {
  if (REL) {
    const uint64_t row = (uint64_t)val * x.d;
    L.template ldf<true>(x.snap + row, pred, it.sv);
    L.ldd(x.mix + row, pred, it.mv);
    it.slot = 0;
    it.w = 0.0;
    return;
  }
  const uint32_t p = val >> x.pshift;
  const uint32_t slot = val & x.smask;
  const bool is_src = slot > x.k;
  LGD_DCHECK(!pred || slot <= x.k + 1, "K4 contribution slot", slot);
  it.slot = slot;
  if (SH && slot == 1) {  // shared negative: its precomputed gradient row (shared.cu SG3)
    it.w = 0.0;
    L.template ldf<true>(x.gneg + (uint64_t)p * x.d, pred, it.sv);
    return;
  }
  // dst (slot 0) uses w = -1: g - IR1 == g + (-1 * IR1) in IEEE arithmetic;
  // TransE's dst coefficient sits after the P x k negative coefficients
  it.w = (pred && slot - 1u < x.k) ? __ldg(x.w + (uint64_t)p * x.k + (slot - 1))
         : (KIND == 3 && pred && slot == 0) ? __ldg(x.w + x.cpos_off + p) : -1.0;
  const uint64_t row = (uint64_t)p * x.d;
  if (IR1 && !SH) {
    // dst / negative: IR1 as K3 formed it; src: mix (both f64 rows)
    L.ldd((is_src ? x.mix : x.ir1) + row, pred, it.mv);
    if (is_src) it.rel = x.rmask ? (val >> x.sbits) & x.rmask : (pred ? __ldg(x.rel_keys + p) : 0);
    return;
  }
  if (KIND != 0)
    it.rel = x.rmask ? (val >> x.sbits) & x.rmask : (pred ? __ldg(x.rel_keys + p) : 0);
  L.template ldf<true>(x.snap + row, pred && !is_src, it.sv);
  L.ldd(x.mix + row, pred && is_src, it.mv);
}

// The first contribution of a K4 v2 segment, staged by cp.async with the
// segment's rows (stage_item): its operand row (snapshot / IR1 / mix /
// shared-negative gradient) at op_s, its weight at w_s.
template <int KIND, int NV, bool SH, bool IR1>
__device__ __forceinline__ void stage_item(const SegCtx& x, const Lanes<KIND, NV>& L, uint32_t val,
                                           uint32_t op_s, uint32_t w_s, int lane) {
  const uint32_t p = val >> x.pshift;
  const uint32_t slot = val & x.smask;
  const uint64_t row = (uint64_t)p * x.d;
  if (SH && slot == 1) {
    L.cpa_s(op_s, x.gneg + row, true);
    return;
  }
  if (lane == 0 && (slot - 1u < x.k || (KIND == 3 && slot == 0))) {
    const double* w = slot == 0 ? x.w + x.cpos_off + p : x.w + (uint64_t)p * x.k + (slot - 1);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(w_s), "l"(w) : "memory");
  }
  if (slot > x.k)
    L.cpd_s(op_s, x.mix + row);
  else if (IR1 && !SH)
    L.cpd_s(op_s, x.ir1 + row);
  else
    L.cpa_s(op_s, x.snap + row, true);
}
// stage_item for the bulk-copy staging (segment_heads of TransE), lane 0
// only: the weight as an 8-byte cp.async, and the operand row's source and
// size for a TMA bulk copy
template <int KIND, bool SH, bool IR1>
__device__ __forceinline__ const void* stage_op_bulk(const SegCtx& x, uint32_t val, uint32_t w_s,
                                                     uint32_t& bytes) {
  const uint32_t p = val >> x.pshift;
  const uint32_t slot = val & x.smask;
  const uint64_t row = (uint64_t)p * x.d;
  if (SH && slot == 1) {
    bytes = x.d * 4;
    return x.gneg + row;
  }
  if (slot - 1u < x.k || (KIND == 3 && slot == 0)) {
    const double* w = slot == 0 ? x.w + x.cpos_off + p : x.w + (uint64_t)p * x.k + (slot - 1);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(w_s), "l"(w) : "memory");
  }
  if (slot > x.k) {
    bytes = x.d * 8;
    return x.mix + row;
  }
  if (IR1 && !SH) {
    bytes = x.d * 8;
    return x.ir1 + row;
  }
  bytes = x.d * 4;
  return x.snap + row;
}

template <int KIND, int NV, bool SH, bool IR1>
__device__ __forceinline__ void load_item_staged(const SegCtx& x, const Lanes<KIND, NV>& L,
                                                 uint32_t val, uint32_t op_s, uint32_t w_s,
                                                 ItemRegs<4 * NV>& it) {
  const uint32_t p = val >> x.pshift;
  const uint32_t slot = val & x.smask;
  const bool is_src = slot > x.k;
  LGD_DCHECK(slot <= x.k + 1, "K4 contribution slot", slot);
  it.slot = slot;
  // (each path fills only the operand add_loaded reads on that path)
  if (SH && slot == 1) {
    it.w = 0.0;
    L.lds_s(op_s, it.sv);
    return;
  }
  double wv = -1.0;
  if (slot - 1u < x.k || (KIND == 3 && slot == 0))
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(wv) : "r"(w_s));
  it.w = wv;
  if (KIND != 0 && (is_src || !IR1 || SH))
    it.rel = x.rmask ? (val >> x.sbits) & x.rmask : __ldg(x.rel_keys + p);
  if (is_src || (IR1 && !SH))
    L.ldd_s(op_s, it.mv);
  else
    L.lds_s(op_s, it.sv);
}

template <int KIND, int NV, bool REL, bool SH, bool IR1 = k4_ir1(KIND), bool R64 = false>
__device__ __forceinline__ void add_loaded(const SegCtx& x, const Lanes<KIND, NV>& L,
                                           const ItemRegs<4 * NV>& it, uint32_t k, double* acc,
                                           const float* own) {
  constexpr int NE = 4 * NV;
  if (SH && !REL && it.slot == 1) {
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] += (double)it.sv[e];
    return;
  }
  if (IR1 && !REL && !SH && it.slot <= k) {  // dst / negative from K3's IR1
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] += KIND == 3 ? it.w * (it.mv[e] - (double)own[e]) : it.w * it.mv[e];
    return;
  }
  // the relation row in FP64: K3's copy (R64) or converted here -- the same
  // values (f32 -> f64 is exact)
  double rv[NE];
  if (KIND != 0 && !REL) {
    if (R64) {
      L.ldd(x.rel64 + (uint64_t)it.rel * x.d, true, rv);
    } else {
      float rf[NE];
      L.template ldf<true>(x.rel_theta + (uint64_t)it.rel * x.d, true, rf);
#pragma unroll
      for (int e = 0; e < NE; ++e) rv[e] = rf[e];
    }
  }
  if (REL || it.slot > k) {  // adj_other(mix): other = src snapshot (REL) or relation row
    double o[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) o[e] = REL ? (double)it.sv[e] : rv[e];
    if (KIND == 2) {
#pragma unroll
      for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int re = 4 * v + t, im = 4 * v + 2 + t;
          const double orr = o[re], ori = o[im], mr = it.mv[re], mi = it.mv[im];
          acc[re] += orr * mr + ori * mi;
          acc[im] += orr * mi - ori * mr;
        }
    } else {
#pragma unroll
      for (int e = 0; e < NE; ++e)
        acc[e] += (KIND == 0 || KIND == 3) ? it.mv[e] : o[e] * it.mv[e];
    }
    return;
  }
  if (KIND == 3) {  // TransE: g += c (u - own row), u = s + r
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const double u = (double)it.sv[e] + rv[e];
      acc[e] += it.w * (u - (double)own[e]);
    }
    return;
  }
  // dst: g -= IR1 (train.cpp:310) as g += (-1) IR1; negative j: g += w_j IR1 (:320)
  if (KIND == 2) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int re = 4 * v + t, im = 4 * v + 2 + t;
        const double sr = it.sv[re], si = it.sv[im], rr = rv[re], ri = rv[im];
        const double xr = sr * rr - si * ri, xi = sr * ri + si * rr;
        acc[re] += it.w * xr;
        acc[im] += it.w * xi;
      }
  } else {
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const double u = KIND == 0 ? (double)it.sv[e] : (double)it.sv[e] * rv[e];
      acc[e] += it.w * u;
    }
  }
}

template <int KIND, int NV, bool REL, bool SH, bool GRAD>
__global__ void __launch_bounds__(kSegThreads, SEG_MINB) segment_pass1_vec(
    BatchArgs a, uint64_t n, const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
    uint32_t* __restrict__ span_list, unsigned int* __restrict__ span_count) {
  constexpr int NE = 4 * NV;
  const int lane = threadIdx.x & 31;
  const uint64_t c = ((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5;
  const uint64_t base = c * 32;
  if (base >= n) return;
  const Lanes<KIND, NV> L(lane, a.dim);
  const SegCtx x{a.snap, a.mix, a.ir1, a.w, a.rel_theta, a.rel_keys, a.dim, a.k,
                 (uint32_t)a.slot_bits, (1u << a.slot_bits) - 1u,
                 (uint32_t)(a.slot_bits + a.rel_bits), a.rel_bits ? (1u << a.rel_bits) - 1u : 0u,
                 a.P * a.k, a.sh_G, nullptr};
  constexpr bool kOwn = KIND == 3 && !REL;  // TransE contributions read the node's own row
  float* __restrict__ theta = REL ? a.rel_theta : a.theta;
  float* __restrict__ state = REL ? a.rel_state : a.state;
  // GRAD: gradients out (lgd_batch_gradients, the relation side pass), no update
  double* gout = GRAD ? (REL ? a.grad_rels : a.grad_nodes) : nullptr;
  const uint64_t d = a.dim;
  const double lr = a.lr, eps = a.eps;
  const uint64_t end = min(base + 32, n);
  const uint64_t i = base + lane;
  const uint32_t key = i < n ? skeys[i] : 0;
  const uint32_t val = i < n ? __ldg(svals + i) : 0;
  const bool head = i < n && (i == 0 || skeys[i - 1] != key);
  const uint32_t hmask = __ballot_sync(0xffffffffu, head);
  const bool cont_in = !(hmask & 1u);
  const bool cont_out = end < n && skeys[end] == skeys[end - 1];
  // lookahead: keys / values of the next chunk
  const uint64_t j = end + lane;
  const uint32_t key2 = (cont_out && j < n) ? skeys[j] : 0;
  const uint32_t val2 = (cont_out && j < n) ? __ldg(svals + j) : 0;
  const uint32_t last_key = __shfl_sync(0xffffffffu, key, (int)(end - base - 1));
  const uint32_t same2 = __ballot_sync(0xffffffffu, cont_out && j < n && key2 == last_key);
  // A segment whose head is in this chunk is "short" when it ends before
  // end + 32 (or at n): this warp finishes it.  The next chunk's warp then
  // skips that leading piece ("lead_done"); both sides use the same rule.
  const int ext = __popc(same2);
  const bool ext_short = cont_out && hmask != 0 && (ext < 32 || end + 32 >= n);
  bool lead_done = false;
  if (cont_in) {
    const bool head_in_prev = skeys[base - 32] != __shfl_sync(0xffffffffu, key, 0);
    lead_done = head_in_prev && (hmask != 0 || end == n);
  }
  const uint32_t smask = hmask | 1u;
  const int np = __popc(smask);
  const int nlive = (int)(end - base);
  auto finishing = [&](int t) {
    return !(t == 0 && cont_in) && !(t == np - 1 && cont_out && !ext_short);
  };
  auto item_val = [&](int q) {  // q may run past the chunk into the lookahead
    const uint32_t v1 = __shfl_sync(0xffffffffu, val, q & 31);
    const uint32_t v2 = __shfl_sync(0xffffffffu, val2, q & 31);
    return q < 32 ? v1 : v2;
  };
  // remaining piece starts, consumed lowest bit first
  uint32_t rest = smask;
  if (lead_done) rest &= rest - 1;
  int t = lead_done ? 1 : 0;
  if (t < np) {
    // row id of every item, lane-parallel once per chunk (pool index -> node)
    const uint32_t myrow = REL ? key : from_pool(a, key);
    auto rowof_at = [&](int s0) { return __shfl_sync(0xffffffffu, myrow, s0 & 31); };
    // theta / state rows of the next kSegDepth pieces are in flight at once:
    // cp.async into this warp's shared-memory ring (no registers held), one
    // commit group per piece.  A piece's first contribution is loaded when the
    // piece is processed (no register prefetch: 64 registers, 32 warps per SM).
    extern __shared__ __align__(16) float seg_ring[];
    const uint32_t rowf = (a.dim + 3) & ~3u;
    const uint32_t slotf = 2 * rowf;  // slot: theta, state
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(seg_ring) +
                          (threadIdx.x >> 5) * kSegDepth * slotf * 4;  // bytes
    const int t0 = t;
    // piece starts still to stage / to process, lowest bit first
    uint32_t srest = rest;
    auto stage = [&](int u, uint32_t slot) {
      if (u < np) {
        const int s0 = __ffs(srest) - 1;
        srest &= srest - 1;
        const uint64_t off = (uint64_t)rowof_at(s0) * d;
        const bool fin = finishing(u) && !gout;
        L.cpa_s(slot, theta + off, fin || kOwn);
        L.cpa_s(slot + rowf * 4, state + off, fin);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int u = 0; u < kSegDepth; ++u) stage(t0 + u, ring + u * slotf * 4);
    uint32_t slot = ring;  // piece t's slot, restaged with piece t + kSegDepth
    int cur = __ffs(rest) - 1;
    rest &= rest - 1;
#pragma unroll 1
    for (; t < np; ++t) {
      K4_TRACE(1);
      const bool has_next = t + 1 < np;
      const int nxt = has_next ? __ffs(rest) - 1 : nlive;
      rest &= rest - 1;
      const int pend = (t == np - 1 && ext_short) ? nlive + ext : nxt;
      ItemRegs<NE> cit;
      load_item<KIND, NV, REL, SH>(x, L, __shfl_sync(0xffffffffu, val, cur), true, cit);
      asm volatile("cp.async.wait_group %0;" ::"n"(kSegDepth - 1) : "memory");
      float th[NE], st[NE];
      L.lds_s(slot, th);
      L.lds_s(slot + rowf * 4, st);
      K4_TRACE(2 + 16 * (pend - cur));
      double acc[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] = 0.0;
      add_loaded<KIND, NV, REL, SH>(x, L, cit, x.k, acc, th);
      K4_TRACE(3);
      for (int q = cur + 1; q < pend; ++q) {
        ItemRegs<NE> it;
        load_item<KIND, NV, REL, SH>(x, L, item_val(q), true, it);
        add_loaded<KIND, NV, REL, SH>(x, L, it, x.k, acc, th);
      }
      K4_TRACE(4);
      const uint32_t row = rowof_at(cur);
      if (t == 0 && cont_in) {
        L.std_(a.part_first + c * d, acc);
      } else if (!finishing(t)) {
        L.std_(a.part_last + c * d, acc);
      } else if (gout) {
        L.std_(gout + (uint64_t)row * d, acc);
        if (lane == 0) (REL ? a.grad_rel_flag : a.grad_node_flag)[row] = 1;
      } else {
        adagrad_lanes(L, acc, th, st, lr, eps);
        K4_TRACE(5);
        L.stf(theta + (uint64_t)row * d, th);
        L.stf(state + (uint64_t)row * d, st);
      }
      stage(t + kSegDepth, slot);  // the slot just read is free again
      slot = slot + slotf * 4 == ring + kSegDepth * slotf * 4 ? ring : slot + slotf * 4;
      cur = nxt;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  if (lane == 0) {
    const int heads = __popc(hmask);
    // pass 2 sees only long segments: a short one ends the chain at this
    // chunk (no kContOut) and its continuation chunk starts "done"
    a.chunk_flags[c] = (heads ? 0 : kNoHead) | ((cont_out && !ext_short) ? kContOut : 0);
    if (heads) atomicAdd(a.counters + (REL ? 1 : 0), (unsigned long long)heads);
    if (heads && cont_out && !ext_short) span_list[atomicAdd(span_count, 1u)] = (uint32_t)c;
  }
}

// One block per chunk that holds the head of a chunk-spanning segment: sum
// part_last[c] and the following chunks' part_first in a fixed order (warp w
// takes chunks w, w + 8, ... in order; warp sums combined in warp order), then
// one Adagrad row update.
template <bool REL>
__global__ void __launch_bounds__(kPass2Threads) segment_pass2(BatchArgs a, uint64_t n,
                                                               const uint32_t* __restrict__ skeys,
                                                               const uint32_t* __restrict__ span_list,
                                                               const unsigned int* __restrict__ span_count) {
  __shared__ double wsum[kPass2Threads / 32][512];
  __shared__ uint32_t s_len;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int W = kPass2Threads / 32;
  const uint32_t d = a.dim;
  const uint64_t nchunks = (n + 31) / 32;
  const unsigned cnt = *span_count;
  for (unsigned idx = blockIdx.x; idx < cnt; idx += gridDim.x) {
    const uint64_t c = span_list[idx];
    if (warp == 0) {  // following chunks covered by the segment, 32 flags per step
      uint32_t L = 0;
      for (uint64_t c0 = c + 1; c0 < nchunks; c0 += 32) {
        const uint64_t c2 = c0 + lane;
        const uint8_t f2 = c2 < nchunks ? a.chunk_flags[c2] : 0;
        const uint32_t stop = __ballot_sync(0xffffffffu, !((f2 & kNoHead) && (f2 & kContOut)));
        if (stop) {
          L += __ffs(stop);
          break;
        }
        L += 32;
      }
      if (lane == 0) s_len = (uint32_t)(L < nchunks - c - 1 ? L : nchunks - c - 1);
    }
    __syncthreads();
    const uint32_t L = s_len;
    for (uint32_t e = lane; e < d; e += 32) {
      double s = 0.0;
      uint32_t q = warp;
      for (; q + 3 * W < L; q += 4 * W) {  // four loads in flight, added in order
        const double v0 = a.part_first[(c + 1 + q) * d + e];
        const double v1 = a.part_first[(c + 1 + q + W) * d + e];
        const double v2 = a.part_first[(c + 1 + q + 2 * W) * d + e];
        const double v3 = a.part_first[(c + 1 + q + 3 * W) * d + e];
        s += v0;
        s += v1;
        s += v2;
        s += v3;
      }
      for (; q < L; q += W) s += a.part_first[(c + 1 + q) * d + e];
      wsum[warp][e] = s;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t kk = skeys[min(c * 32 + 32, n) - 1];
      const uint32_t row = REL ? kk : from_pool(a, kk);
      double* gout = REL ? a.grad_rels : a.grad_nodes;
      float* th = row_theta<REL>(a, row);
      float* st = row_state<REL>(a, row);
      for (uint32_t e = lane; e < d; e += 32) {
        double gsum = a.part_last[c * d + e];
        for (int w = 0; w < W; ++w) gsum += wsum[w][e];
        if (gout) {
          gout[(size_t)row * d + e] = gsum;
        } else {
          float tv = th[e], sv = st[e];
          adagrad_elem(gsum, tv, sv, a.lr, a.eps);
          th[e] = tv;
          st[e] = sv;
        }
      }
      if (gout && lane == 0) (REL ? a.grad_rel_flag : a.grad_node_flag)[row] = 1;
    }
    __syncthreads();
  }
}

// ------------------------------------------ K4 v2: whole-segment updates
// Every segment (one unique node's sorted contributions) is summed by ONE
// warp, sequentially in FP64 in the reference's std::map order
// (train.cpp:290-333), then its row gets the Adagrad update
// (train.cpp:342-354); no partial sums cross warps for segments of up to
// kLongSeg items.
//   segment_heads  warp per 32 sorted items of the batch: it owns the segments
//                  whose HEAD lies in its items.  Head and terminator masks of
//                  its items and the next 32 (two ballots) give every owned
//                  segment's length; a segment of <= kLongSeg items ends inside
//                  that window, so the warp finishes it.  The theta / state
//                  rows of the next kSegDepth segments are in flight in the
//                  warp's cp.async ring; payloads come from two 32-item
//                  register windows.  No continuation pieces, no second pass.
//   long_chunks /  segments of more than kLongSeg items (hubs: up to thousands
//   long_combine   of contributions per batch under the power law) are listed
//                  once per bucket (launch_long_list), cut into 32-item chunks
//                  summed by independent warps, and their partials added in
//                  chunk order (deterministic) by one warp per segment.  They
//                  run on the side stream, concurrently with segment_heads
//                  (disjoint rows).
// No atomics on rows; every row is written by exactly one warp.
constexpr uint32_t kLongSeg = 32;

// ring slot of a segment (bytes): theta row, state row, the first
// contribution's operand row (f64 width), its weight
__host__ __device__ constexpr uint32_t seg_slot_bytes(uint32_t rowf) { return 16 * rowf + 16; }

// TransE's K4 runs faster with 80 registers (3 blocks of 256 per SM) than with
// 64 (4 blocks): Friendster K4 0.907 -> 0.860 ms; the other models are best
// at 64 (TW DistMult 0.80 vs 0.82, LJ Dot 0.49 vs 0.51, FM ComplEx 0.69 vs 0.70
// ms; profiles/r02zh, r02zi)
template <int KIND>
constexpr int seg_heads_minb() { return KIND == 3 && SEG_MINB == 4 ? 3 : SEG_MINB; }
// segment_heads' ring depth per model: 3 for Dot / ComplEx (LJ K4 0.499 ->
// 0.489 ms, FM 0.686 -> 0.683), 2 for DistMult / TransE (TW 0.80 vs 0.81,
// Friendster 0.866 vs 0.884; profiles/r02m, r02zk); -DSEG_DEPTH_FIXED: SEG_DEPTH for all
template <int KIND>
constexpr int seg_heads_depth() {
#ifdef SEG_DEPTH_FIXED
  return SEG_DEPTH;
#else
  return KIND == 0 || KIND == 2 ? 3 : 2;
#endif
}

template <int KIND, int NV, bool SH, bool IR1, bool R64>
__global__ void __launch_bounds__(kSegThreads, seg_heads_minb<KIND>()) segment_heads(
    BatchArgs a, const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
    uint64_t b0, uint64_t b1) {
  constexpr int NE = 4 * NV;
  const int lane = threadIdx.x & 31;
  const uint64_t base = b0 + (((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5) * 32;
  if (base >= b1) return;
  const Lanes<KIND, NV> L(lane, a.dim);
  const SegCtx x{a.snap, a.mix, a.ir1, a.w, a.rel_theta, a.rel_keys, a.dim, a.k,
                 (uint32_t)a.slot_bits, (1u << a.slot_bits) - 1u,
                 (uint32_t)(a.slot_bits + a.rel_bits), a.rel_bits ? (1u << a.rel_bits) - 1u : 0u,
                 a.P * a.k, a.sh_G, a.rel64};
  float* __restrict__ theta = a.theta;
  float* __restrict__ state = a.state;
  const uint64_t d = a.dim;
  const double lr = a.lr, eps = a.eps;
  // head / terminator masks of items [base, base + 64): the batch ends at b1
  const uint64_t i = base + lane, j = i + 32;
  const uint32_t key = i < b1 ? __ldg(skeys + i) : 0u;
  const uint32_t key2 = j < b1 ? __ldg(skeys + j) : 0u;
  const uint32_t prev = (i < b1 && i > b0) ? __ldg(skeys + i - 1) : ~key;
  const uint32_t prev2 = __shfl_sync(0xffffffffu, key, 31);  // item base + 31
  const uint32_t prev2_l = __shfl_up_sync(0xffffffffu, key2, 1);
  const bool head = i < b1 && key != prev;
  const bool term2 = j >= b1 || key2 != (lane ? prev2_l : prev2);
  const uint32_t hmask = __ballot_sync(0xffffffffu, head);
  const uint32_t tmask0 = __ballot_sync(0xffffffffu, head || i >= b1);
  const uint32_t tmask1 = __ballot_sync(0xffffffffu, term2);
  const uint64_t ends = (uint64_t)tmask0 | ((uint64_t)tmask1 << 32);
  if (lane == 0 && hmask) atomicAdd(a.counters, (unsigned long long)__popc(hmask));
  // lane l with a head: segment length (0 = long, left to the long path)
  uint32_t my_len = 0;
  if (head) {
    const uint64_t above = ends & ~((2ull << lane) - 1);  // terminators after the head
    const uint32_t e = above ? (uint32_t)__ffsll((long long)above) - 1 : 64u;
    my_len = e - lane <= kLongSeg ? e - lane : 0u;
  }
  uint32_t todo = __ballot_sync(0xffffffffu, my_len != 0);
  if (!todo) return;
  const uint32_t my_row = my_len ? from_pool(a, key) : 0u;
  LGD_DCHECK(!my_len || (my_row < a.num_nodes && my_len <= kLongSeg && base + lane + my_len <= b1),
             "K4 segment outside the batch / table", my_row);
  const uint32_t w0 = i < b1 ? __ldg(svals + i) : 0u;
  const uint32_t w1 = j < b1 ? __ldg(svals + j) : 0u;
  auto item = [&](uint32_t o) {  // o < 64: the item at base + o
    const uint32_t v0 = __shfl_sync(0xffffffffu, w0, o & 31);
    const uint32_t v1 = __shfl_sync(0xffffffffu, w1, o & 31);
    return o < 32 ? v0 : v1;
  };
  // ring of kDepth slots per warp: the theta / state rows AND the first
  // contribution's operand row and weight of the next segments are in flight
  // (cp.async, one commit group per segment), so a segment starts without a
  // dependent global load
  constexpr int kDepth = seg_heads_depth<KIND>();
  extern __shared__ __align__(16) float seg_ring[];
  const uint32_t rowf = (a.dim + 3) & ~3u;
  const uint32_t sb = seg_slot_bytes(rowf);
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(seg_ring) +
                        (threadIdx.x >> 5) * kDepth * sb;  // bytes
  uint32_t srest = todo;  // segments still to stage, lowest first
  // TransE stages its rows as TMA bulk copies issued by one lane (one
  // mbarrier per ring slot, after all warps' rings): Friendster K4 0.870 ->
  // 0.829 ms; at the 64-register cap of the other models the variant spills
  // (TW -17%, LJ -21%, FM -2%; profiles/r02zy, r02zz; -DK4_BULK_ALL=1 builds that A/B)
  constexpr bool kBulk = K4_BULK_ALL || KIND == 3;
  const uint32_t bars = (uint32_t)__cvta_generic_to_shared(seg_ring) +
                        (kSegThreads / 32) * kDepth * sb + (threadIdx.x >> 5) * kDepth * 8;
  if constexpr (kBulk) {
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < kDepth; ++u) mbar_init_s(bars + 8 * u, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  auto stage = [&](uint32_t u) {  // ring slot u
    const uint32_t slot = ring + u * sb;
    if (srest) {
      const int h = __ffs(srest) - 1;
      srest &= srest - 1;
      const uint64_t off = (uint64_t)__shfl_sync(0xffffffffu, my_row, h) * d;
      if constexpr (kBulk) {  // three bulk copies from lane 0, tracked by the slot's mbarrier
        const uint32_t v = item(h);
        if (lane == 0) {
          const uint32_t rb = (uint32_t)d * 4;
          uint32_t ob;
          const void* op = stage_op_bulk<KIND, SH, IR1>(x, v, slot + 16 * rowf, ob);
          mbar_expect_s(bars + 8 * u, 2 * rb + ob);
          const uint32_t dst[3] = {slot, slot + rowf * 4, slot + 8 * rowf};
          const void* src[3] = {theta + off, state + off, op};
          const uint32_t len[3] = {rb, rb, ob};
#pragma unroll
          for (int c = 0; c < 3; ++c)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                "[%3];" ::"r"(dst[c]),
                "l"(src[c]), "r"(len[c]), "r"(bars + 8 * u)
                : "memory");
        }
      } else {
        L.cpa_s(slot, theta + off, true);
        L.cpa_s(slot + rowf * 4, state + off, true);
        stage_item<KIND, NV, SH, IR1>(x, L, item(h), slot + 8 * rowf, slot + 16 * rowf, lane);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
#pragma unroll
  for (int u = 0; u < kDepth; ++u) stage(u);
  uint32_t u = 0, ph = 0;  // the slot being consumed and its mbarrier phase
#pragma unroll 1
  while (todo) {
    const int h = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint32_t len = __shfl_sync(0xffffffffu, my_len, h);
    const uint32_t row = __shfl_sync(0xffffffffu, my_row, h);
    const uint32_t v0 = item(h);
    asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    if constexpr (kBulk) mbar_wait_s(bars + 8 * u, ph);
    const uint32_t slot = ring + u * sb;
    __syncwarp();  // lane 0 staged the weight every lane reads
    float th[NE], st[NE];
    L.lds_s(slot, th);
    L.lds_s(slot + rowf * 4, st);
    ItemRegs<NE> cit;
    load_item_staged<KIND, NV, SH, IR1>(x, L, v0, slot + 8 * rowf, slot + 16 * rowf, cit);
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
    add_loaded<KIND, NV, false, SH, IR1, R64>(x, L, cit, x.k, acc, th);
    for (uint32_t q = h + 1; q < h + len; ++q) {
      ItemRegs<NE> it;
      load_item<KIND, NV, false, SH, IR1>(x, L, item(q), true, it);
      add_loaded<KIND, NV, false, SH, IR1, R64>(x, L, it, x.k, acc, th);
    }
    adagrad_lanes(L, acc, th, st, lr, eps);
    L.stf(theta + (uint64_t)row * d, th);
    L.stf(state + (uint64_t)row * d, st);
    __syncwarp();  // every lane read the weight before the slot is restaged
    stage(u);  // the slot just read is free again
    if (++u == kDepth) {
      u = 0;
      ph ^= 1;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// ------------------------------- K4 v4: flattened whole-segment updates
// The warp owns the segments whose heads lie in its 32 sorted items (as
// segment_heads) but walks them as ONE flat sequence of 16-byte row vectors:
// at each step lane l takes vector f = 32 s + l of the concatenated rows of
// the warp's segments (d = 100: 25 vectors per row), so every lane works --
// no idle lanes at row ends -- and the per-segment bookkeeping is paid once
// per 32 vectors, not once per row.  A lane sums its vector's contributions
// sequentially in the reference order (all lanes step through the longest
// segment of the step, predicated), runs the Adagrad update on its four
// elements and stores them.  theta / state and the operands are plain
// coalesced 16-byte loads: consecutive lanes read consecutive vectors of the
// same row.
template <int KIND, bool SH, bool IR1, bool R64>
__global__ void __launch_bounds__(kSegThreads, SEG_MINB) segment_flat(
    BatchArgs a, const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
    uint64_t b0, uint64_t b1) {
  const int lane = threadIdx.x & 31;
  const uint64_t base = b0 + (((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5) * 32;
  if (base >= b1) return;
  const SegCtx x{a.snap, a.mix, a.ir1, a.w, a.rel_theta, a.rel_keys, a.dim, a.k,
                 (uint32_t)a.slot_bits, (1u << a.slot_bits) - 1u,
                 (uint32_t)(a.slot_bits + a.rel_bits), a.rel_bits ? (1u << a.rel_bits) - 1u : 0u,
                 a.P * a.k, a.sh_G, a.rel64};
  const uint64_t d = a.dim;
  const double lr = a.lr, eps = a.eps;
  const uint64_t i = base + lane, j = i + 32;
  const uint32_t key = i < b1 ? __ldg(skeys + i) : 0u;
  const uint32_t key2 = j < b1 ? __ldg(skeys + j) : 0u;
  const uint32_t prev = (i < b1 && i > b0) ? __ldg(skeys + i - 1) : ~key;
  const uint32_t prev2 = __shfl_sync(0xffffffffu, key, 31);
  const uint32_t prev2_l = __shfl_up_sync(0xffffffffu, key2, 1);
  const bool head = i < b1 && key != prev;
  const bool term2 = j >= b1 || key2 != (lane ? prev2_l : prev2);
  const uint32_t hmask = __ballot_sync(0xffffffffu, head);
  const uint32_t tmask0 = __ballot_sync(0xffffffffu, head || i >= b1);
  const uint32_t tmask1 = __ballot_sync(0xffffffffu, term2);
  const uint64_t ends = (uint64_t)tmask0 | ((uint64_t)tmask1 << 32);
  if (lane == 0 && hmask) atomicAdd(a.counters, (unsigned long long)__popc(hmask));
  uint32_t my_len = 0;
  if (head) {
    const uint64_t above = ends & ~((2ull << lane) - 1);
    const uint32_t e = above ? (uint32_t)__ffsll((long long)above) - 1 : 64u;
    my_len = e - lane <= kLongSeg ? e - lane : 0u;
  }
  const uint32_t todo = __ballot_sync(0xffffffffu, my_len != 0);
  if (!todo) return;
  const int ns = __popc(todo);
  const uint32_t my_row = my_len ? from_pool(a, key) : 0u;
  LGD_DCHECK(!my_len || (my_row < a.num_nodes && base + lane + my_len <= b1),
             "K4 segment outside the batch / table", my_row);
  // compact: lane c holds the c-th short segment (head position, length, row)
  uint32_t m = todo;  // lane c: the c-th set bit of todo
  for (int t = 0; t < lane && m; ++t) m &= m - 1;
  const int sl = m ? __ffs(m) - 1 : 0;
  const uint32_t c_pos = __shfl_sync(0xffffffffu, (uint32_t)lane, sl);
  const uint32_t c_len = __shfl_sync(0xffffffffu, my_len, sl);
  const uint32_t c_row = __shfl_sync(0xffffffffu, my_row, sl);
  const uint32_t w0 = i < b1 ? __ldg(svals + i) : 0u;
  const uint32_t w1 = j < b1 ? __ldg(svals + j) : 0u;
  const uint32_t nvec = KIND == 2 ? (uint32_t)(d / 4) : (uint32_t)(d / 4);  // 16-byte vectors per row
  const uint32_t total = (uint32_t)ns * nvec;
  // this lane's (segment, vector) at flat index lane, advanced by 32 per step;
  // the next step's theta / state vectors are loaded while this step sums
  uint32_t seg = 0, q = lane;
  while (q >= nvec) {
    q -= nvec;
    ++seg;
  }
  auto row_of = [&](uint32_t sgv) { return __shfl_sync(0xffffffffu, c_row, (int)sgv & 31); };
  float th[4], st[4];
  {
    const bool act0 = lane < total;
    const uint32_t r0 = row_of(act0 ? seg : 0);
    const Lanes<KIND, 1> L0(act0 ? (int)q : 0, a.dim);
    L0.template ldf<false>(a.theta + (uint64_t)r0 * d, act0, th);
    L0.template ldf<false>(a.state + (uint64_t)r0 * d, act0, st);
  }
#pragma unroll 1
  for (uint32_t f0 = 0; f0 < total; f0 += 32) {
    const bool act = f0 + lane < total;
    const int sg = act ? (int)seg : 0;
    // (every lane takes part in each shuffle: none sits under a condition)
    const uint32_t pos = __shfl_sync(0xffffffffu, c_pos, sg);
    const uint32_t len_s = __shfl_sync(0xffffffffu, c_len, sg);
    const uint32_t row = __shfl_sync(0xffffffffu, c_row, sg);
    const uint32_t len = act ? len_s : 0u;
    const Lanes<KIND, 1> L(act ? (int)q : 0, a.dim);
    const uint64_t off = (uint64_t)row * d;
    // the next step's position and rows, in flight during this step
    uint32_t nseg = seg, nq = q + 32;
    while (nq >= nvec) {
      nq -= nvec;
      ++nseg;
    }
    const bool nact = f0 + 32 + lane < total;
    const uint32_t nrow = row_of(nact ? nseg : 0);
    float nth[4], nst[4];
    {
      const Lanes<KIND, 1> Ln(nact ? (int)nq : 0, a.dim);
      Ln.template ldf<false>(a.theta + (uint64_t)nrow * d, nact, nth);
      Ln.template ldf<false>(a.state + (uint64_t)nrow * d, nact, nst);
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t maxlen = len;
#pragma unroll
    for (int o = 16; o; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    for (uint32_t t = 0; t < maxlen; ++t) {  // contributions in order; lanes past their end idle
      const uint32_t o = pos + (t < len ? t : 0u);
      const uint32_t v0 = __shfl_sync(0xffffffffu, w0, o & 31);
      const uint32_t v1 = __shfl_sync(0xffffffffu, w1, o & 31);
      if (t < len) {
        ItemRegs<4> it;
        load_item<KIND, 1, false, SH, IR1>(x, L, o < 32 ? v0 : v1, true, it);
        add_loaded<KIND, 1, false, SH, IR1, R64>(x, L, it, x.k, acc, th);
      }
    }
    if (act) {
      adagrad_lanes(L, acc, th, st, lr, eps);
      L.stf(a.theta + off, th);
      L.stf(a.state + off, st);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      th[e] = nth[e];
      st[e] = nst[e];
    }
    seg = nseg;
    q = nq;
  }
}

// --------------------------- K4 v3: warp-specialised whole-segment updates
// The same segments as segment_heads (<= kLongSeg contributions, summed whole
// in the reference order), split between producer and consumer warps so
// neither carries the other's registers or bookkeeping:
//   producer warps  decode 32 sorted items at a time lane-parallel (heads,
//                   lengths, rows, first payloads) and stage each segment into
//                   a consumer's ring slot with cp.async: its theta / state
//                   rows, its first contribution's operand row and weight, and
//                   its metadata; completion is tracked by the slot's mbarrier
//                   (cp.async.mbarrier.arrive.noinc), so the producer never
//                   waits for its copies;
//   consumer warps  wait on the slot, sum the contributions (the first from
//                   shared memory, any others from global), run the Adagrad
//                   row update, store the row and release the slot.
// Block: kWsProducers producers, kWsConsumers consumers (each producer feeds
// its own kWsConsumers / kWsProducers), kWsDepth slots per consumer.
#ifndef WS_PRODUCERS
#define WS_PRODUCERS 4
#endif
#ifndef WS_BULK  // 1: producers stage a segment with three TMA bulk copies from one lane
#define WS_BULK 1
#endif
constexpr int kWsProducers = WS_PRODUCERS;
constexpr int kWsConsumers = 8;
constexpr int kWsDepth = 3;
constexpr int kWsThreads = (kWsProducers + kWsConsumers) * 32;
constexpr int kWsPer = kWsConsumers / kWsProducers;
constexpr uint32_t kWsChunks = 64;  // 32-item chunks per block
// slot (bytes): theta 4 rowf | state 4 rowf | operand 8 rowf | weight 8 | meta 16
__host__ __device__ constexpr uint32_t ws_slot_bytes(uint32_t rowf) { return 16 * rowf + 32; }
__host__ __device__ constexpr uint32_t ws_bar_bytes() { return 2 * kWsConsumers * kWsDepth * 8; }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cpasync(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
// waits with a back-off so a waiting warp does not take issue slots from the
// warps doing work
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  if (mbar_try_wait(bar, phase)) return;
  uint32_t ns = 32;
  while (!mbar_try_wait(bar, phase)) {
    __nanosleep(ns);
    ns = ns < 256 ? 2 * ns : ns;
  }
}

template <int KIND, int NV, bool SH, bool IR1, bool R64>
__global__ void __launch_bounds__(kWsThreads, 2) segment_ws(
    BatchArgs a, const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
    uint64_t b0, uint64_t b1) {
  constexpr int NE = 4 * NV;
  extern __shared__ __align__(16) unsigned char ws_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(ws_smem);  // [consumer][slot]
  uint64_t* empty = full + kWsConsumers * kWsDepth;
  const uint32_t rowf = (a.dim + 3) & ~3u;
  const uint32_t sb = ws_slot_bytes(rowf);
  const uint32_t slots = (uint32_t)__cvta_generic_to_shared(ws_smem) + ws_bar_bytes();
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsConsumers * kWsDepth; ++i) {
      // bulk staging: lane 0's expect-tx arrive + its cp.async (weight) arrive;
      // else 32 producer lanes' copies + the metadata arrive
      mbar_init(full + i, WS_BULK ? 2 : 33);
      mbar_init(empty + i, 1);  // the consumer's release
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < kWsConsumers * kWsDepth; ++i) mbar_arrive(empty + i);  // slots start free
  }
  __syncthreads();
  const Lanes<KIND, NV> L(lane, a.dim);
  const SegCtx x{a.snap, a.mix, a.ir1, a.w, a.rel_theta, a.rel_keys, a.dim, a.k,
                 (uint32_t)a.slot_bits, (1u << a.slot_bits) - 1u,
                 (uint32_t)(a.slot_bits + a.rel_bits), a.rel_bits ? (1u << a.rel_bits) - 1u : 0u,
                 a.P * a.k, a.sh_G, a.rel64};
  const uint64_t d = a.dim;
  auto slot_addr = [&](int c, int s) { return slots + (uint32_t)(c * kWsDepth + s) * sb; };
  if (warp < kWsProducers) {
    // ----------------------------------------------------------- producer
    const uint64_t cb0 = b0 + (uint64_t)blockIdx.x * kWsChunks * 32;
    const uint64_t cb1 = min(b1, cb0 + (uint64_t)kWsChunks * 32);
    uint32_t state = 0;  // per own consumer: use count mod 2 kWsDepth, 3 bits each
    int rr = 0;          // next own consumer
    auto claim = [&](int& c, uint32_t& sa, uint32_t& par) {
      const uint32_t st = (state >> (3 * rr)) & 7u;
      c = warp * kWsPer + rr;
      const int s = (int)(st % kWsDepth);
      par = st / kWsDepth;
      state = (state & ~(7u << (3 * rr))) | (((st + 1) % (2 * kWsDepth)) << (3 * rr));
      rr = (rr + 1) % kWsPer;
      mbar_wait(empty + c * kWsDepth + s, par);
      sa = slot_addr(c, s);
      return s;
    };
    for (uint64_t base = cb0 + (uint64_t)warp * 32; base < cb1; base += kWsProducers * 32) {
      const uint64_t i = base + lane, j = i + 32;
      const uint32_t key = i < b1 ? __ldg(skeys + i) : 0u;
      const uint32_t key2 = j < b1 ? __ldg(skeys + j) : 0u;
      const uint32_t prev = (i < b1 && i > b0) ? __ldg(skeys + i - 1) : ~key;
      const uint32_t prev2 = __shfl_sync(0xffffffffu, key, 31);
      const uint32_t prev2_l = __shfl_up_sync(0xffffffffu, key2, 1);
      const bool head = i < b1 && key != prev;
      const bool term2 = j >= b1 || key2 != (lane ? prev2_l : prev2);
      const uint32_t hmask = __ballot_sync(0xffffffffu, head);
      const uint32_t tmask0 = __ballot_sync(0xffffffffu, head || i >= b1);
      const uint32_t tmask1 = __ballot_sync(0xffffffffu, term2);
      const uint64_t ends = (uint64_t)tmask0 | ((uint64_t)tmask1 << 32);
      if (lane == 0 && hmask) atomicAdd(a.counters, (unsigned long long)__popc(hmask));
      uint32_t my_len = 0;
      if (head) {
        const uint64_t above = ends & ~((2ull << lane) - 1);
        const uint32_t e = above ? (uint32_t)__ffsll((long long)above) - 1 : 64u;
        my_len = e - lane <= kLongSeg ? e - lane : 0u;
      }
      uint32_t todo = __ballot_sync(0xffffffffu, my_len != 0);
      const uint32_t my_row = my_len ? from_pool(a, key) : 0u;
      const uint32_t my_val = i < b1 ? __ldg(svals + i) : 0u;  // a head's own first item
      LGD_DCHECK(!my_len || (my_row < a.num_nodes && base + lane + my_len <= b1),
                 "K4 segment outside the batch / table", my_row);
      while (todo) {
        const int h = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t row = __shfl_sync(0xffffffffu, my_row, h);
        const uint32_t val = __shfl_sync(0xffffffffu, my_val, h);
        const uint32_t len = __shfl_sync(0xffffffffu, my_len, h);
        int c;
        uint32_t sa, par;
        const int s = claim(c, sa, par);
        const uint64_t off = (uint64_t)row * d;
        if (WS_BULK) {  // lane 0: three TMA bulk copies on the slot's full barrier
          if (lane == 0) {
            const uint32_t fb = smem_addr(full + c * kWsDepth + s);
            const uint32_t rb = (uint32_t)d * 4;
            uint32_t ob;
            const void* op = stage_op_bulk<KIND, SH, IR1>(x, val, sa + 16 * rowf, ob);
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sa + 16 * rowf + 16),
                         "r"(row), "r"(len), "r"((uint32_t)(base + h)), "r"(val)
                         : "memory");
            mbar_expect_s(fb, 2 * rb + ob);
            const uint32_t dst[3] = {sa, sa + 4 * rowf, sa + 8 * rowf};
            const void* src[3] = {a.theta + off, a.state + off, op};
            const uint32_t len3[3] = {rb, rb, ob};
#pragma unroll
            for (int q = 0; q < 3; ++q)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                  "%2, [%3];" ::"r"(dst[q]),
                  "l"(src[q]), "r"(len3[q]), "r"(fb)
                  : "memory");
            mbar_arrive_cpasync(full + c * kWsDepth + s);  // the weight's cp.async
          }
        } else {
          L.cpa_s(sa, a.theta + off, true);
          L.cpa_s(sa + 4 * rowf, a.state + off, true);
          stage_item<KIND, NV, SH, IR1>(x, L, val, sa + 8 * rowf, sa + 16 * rowf, lane);
          if (lane == 0) {
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sa + 16 * rowf + 16),
                         "r"(row), "r"(len), "r"((uint32_t)(base + h)), "r"(val)
                         : "memory");
            mbar_arrive(full + c * kWsDepth + s);
          }
          mbar_arrive_cpasync(full + c * kWsDepth + s);
        }
      }
    }
    for (int t = 0; t < kWsPer; ++t) {  // end of work: a zero-length slot per consumer
      int c;
      uint32_t sa, par;
      const int s = claim(c, sa, par);
      if (lane == 0) {
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sa + 16 * rowf + 16),
                     "r"(0u), "r"(0u), "r"(0u), "r"(0u)
                     : "memory");
        mbar_arrive(full + c * kWsDepth + s);
        if (WS_BULK) mbar_arrive_cpasync(full + c * kWsDepth + s);
      }
      if (!WS_BULK) mbar_arrive_cpasync(full + c * kWsDepth + s);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  // ------------------------------------------------------------- consumer
  const int c = warp - kWsProducers;
  const double lr = a.lr, eps = a.eps;
  for (uint32_t k = 0;; ++k) {
    const int s = (int)(k % kWsDepth);
    mbar_wait(full + c * kWsDepth + s, (k / kWsDepth) & 1u);
    const uint32_t sa = slot_addr(c, s);
    uint32_t row, len, q0, val;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(row), "=r"(len), "=r"(q0), "=r"(val)
                 : "r"(sa + 16 * rowf + 16));
    if (len == 0) break;
    float th[NE], st[NE];
    L.lds_s(sa, th);
    L.lds_s(sa + 4 * rowf, st);
    ItemRegs<NE> cit;
    load_item_staged<KIND, NV, SH, IR1>(x, L, val, sa + 8 * rowf, sa + 16 * rowf, cit);
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
    add_loaded<KIND, NV, false, SH, IR1, R64>(x, L, cit, x.k, acc, th);
    for (uint32_t q = q0 + 1; q < q0 + len; ++q) {
      ItemRegs<NE> it;
      load_item<KIND, NV, false, SH, IR1>(x, L, __ldg(svals + q), true, it);
      add_loaded<KIND, NV, false, SH, IR1, R64>(x, L, it, x.k, acc, th);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + c * kWsDepth + s);  // slot read: release it
    adagrad_lanes(L, acc, th, st, lr, eps);
    L.stf(a.theta + (uint64_t)row * d, th);
    L.stf(a.state + (uint64_t)row * d, st);
  }
}

// The bucket's long segments (launch_long_list): head item, end item,
// exclusive prefix of their 32-item chunk counts, first long segment of each
// batch.  Chunk c of long segment j covers items head + 32 (c - base[j]) + [0, 32).
struct LongList {
  const uint32_t* head;
  const uint32_t* end;
  const uint32_t* chunk_base;
  const uint32_t* first;  // nb + 1 entries
};

template <int KIND, int NV, bool SH, bool IR1, bool R64>
__global__ void __launch_bounds__(kSegThreads) long_chunks(
    BatchArgs a, const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals,
    LongList ll, uint32_t batch, double* __restrict__ part) {
  constexpr int NE = 4 * NV;
  const int lane = threadIdx.x & 31;
  const uint32_t lf = ll.first[batch], le = ll.first[batch + 1];
  if (lf == le) return;
  const Lanes<KIND, NV> L(lane, a.dim);
  const SegCtx x{a.snap, a.mix, a.ir1, a.w, a.rel_theta, a.rel_keys, a.dim, a.k,
                 (uint32_t)a.slot_bits, (1u << a.slot_bits) - 1u,
                 (uint32_t)(a.slot_bits + a.rel_bits), a.rel_bits ? (1u << a.rel_bits) - 1u : 0u,
                 a.P * a.k, a.sh_G, a.rel64};
  const uint32_t c0 = ll.chunk_base[lf], c1 = ll.chunk_base[le];
  const uint64_t d = a.dim;
  const uint32_t nwarps = gridDim.x * (kSegThreads / 32);
  for (uint32_t c = c0 + blockIdx.x * (kSegThreads / 32) + (threadIdx.x >> 5); c < c1; c += nwarps) {
    uint32_t lo = lf, hi = le;  // last j with chunk_base[j] <= c
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(ll.chunk_base + mid) <= c) lo = mid; else hi = mid;
    }
    const uint32_t s0 = __ldg(ll.head + lo), s1 = __ldg(ll.end + lo);
    const uint32_t q0 = s0 + 32 * (c - __ldg(ll.chunk_base + lo));
    const uint32_t q1 = min(q0 + 32, s1);
    LGD_DCHECK(q0 < q1 && s1 - s0 > kLongSeg, "long segment chunk", q0);
    const uint32_t w = q0 + lane < q1 ? __ldg(svals + q0 + lane) : 0u;
    float own[NE];
    if (KIND == 3) {  // TransE contributions read the node's own (pre-update) row
      const uint32_t row = from_pool(a, __ldg(skeys + s0));
      L.template ldf<true>(a.theta + (uint64_t)row * d, true, own);
    }
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
    for (uint32_t q = q0; q < q1; ++q) {
      ItemRegs<NE> it;
      load_item<KIND, NV, false, SH, IR1>(x, L, __shfl_sync(0xffffffffu, w, q - q0), true, it);
      add_loaded<KIND, NV, false, SH, IR1, R64>(x, L, it, x.k, acc, own);
    }
    L.std_(part + (uint64_t)(c - c0) * d, acc);
  }
}

template <int KIND, int NV>
__global__ void __launch_bounds__(kSegThreads) long_combine(
    BatchArgs a, const uint32_t* __restrict__ skeys, LongList ll, uint32_t batch,
    const double* __restrict__ part) {
  constexpr int NE = 4 * NV;
  const int lane = threadIdx.x & 31;
  const uint32_t lf = ll.first[batch], le = ll.first[batch + 1];
  if (lf == le) return;
  const Lanes<KIND, NV> L(lane, a.dim);
  const uint32_t c0 = ll.chunk_base[lf];
  const uint64_t d = a.dim;
  const uint32_t nwarps = gridDim.x * (kSegThreads / 32);
  for (uint32_t j = lf + blockIdx.x * (kSegThreads / 32) + (threadIdx.x >> 5); j < le; j += nwarps) {
    const uint32_t row = from_pool(a, __ldg(skeys + __ldg(ll.head + j)));
    const uint32_t b0 = __ldg(ll.chunk_base + j) - c0, b1 = __ldg(ll.chunk_base + j + 1) - c0;
    double acc[NE];
    L.ldd(part + (uint64_t)b0 * d, true, acc);
    uint32_t c = b0 + 1;
    for (; c + 4 <= b1; c += 4) {  // four partials in flight, added in chunk order
      double v0[NE], v1[NE], v2[NE], v3[NE];
      L.ldd(part + (uint64_t)c * d, true, v0);
      L.ldd(part + (uint64_t)(c + 1) * d, true, v1);
      L.ldd(part + (uint64_t)(c + 2) * d, true, v2);
      L.ldd(part + (uint64_t)(c + 3) * d, true, v3);
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] = (((acc[e] + v0[e]) + v1[e]) + v2[e]) + v3[e];
    }
    for (; c < b1; ++c) {
      double v[NE];
      L.ldd(part + (uint64_t)c * d, true, v);
#pragma unroll
      for (int e = 0; e < NE; ++e) acc[e] += v[e];
    }
    float th[NE], st[NE];
    L.template ldf<false>(a.theta + (uint64_t)row * d, true, th);
    L.template ldf<false>(a.state + (uint64_t)row * d, true, st);
    adagrad_lanes(L, acc, th, st, a.lr, a.eps);
    L.stf(a.theta + (uint64_t)row * d, th);
    L.stf(a.state + (uint64_t)row * d, st);
  }
}

// heads of segments longer than kLongSeg: the item 32 places on has the same key
struct LongHead {
  const uint32_t* keys;
  uint64_t n;
  __host__ __device__ __forceinline__ bool operator()(const uint32_t& i) const {
    return (i == 0 || keys[i] != keys[i - 1]) && i + kLongSeg < n && keys[i + kLongSeg] == keys[i];
  }
};

// One block: each long segment's end (galloping search for the first item
// with another key), chunk_base = exclusive prefix of the chunk counts,
// first[b] = first long segment at or after batch b's first item.
__global__ void __launch_bounds__(1024) long_index_kernel(
    const uint32_t* __restrict__ keys, uint64_t n, const uint32_t* __restrict__ head,
    const uint32_t* __restrict__ nlong_p, uint64_t batch_items, uint32_t nb,
    uint32_t* __restrict__ end, uint32_t* __restrict__ chunk_base, uint32_t* __restrict__ first) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t carry;
  const uint32_t nlong = *nlong_p;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t t0 = 0; t0 <= nlong; t0 += 1024) {
    const uint32_t jj = t0 + threadIdx.x;
    uint32_t c = 0;
    if (jj < nlong) {
      const uint64_t h = head[jj];
      const uint32_t k = keys[h];
      uint64_t lo = h + kLongSeg, step = 64;  // keys[lo] == k
      uint64_t hi = lo + step;
      while (hi < n && keys[hi] == k) {
        lo = hi;
        step *= 2;
        hi = lo + step;
      }
      if (hi > n) hi = n;
      while (hi - lo > 1) {  // keys[lo] == k, keys[hi] != k (or hi == n)
        const uint64_t mid = (lo + hi) >> 1;
        if (keys[mid] == k) lo = mid; else hi = mid;
      }
      end[jj] = (uint32_t)hi;
      c = (uint32_t)((hi - h + 31) / 32);
    }
    uint32_t ex, total;
    Scan(tmp).ExclusiveSum(c, ex, total);
    if (jj <= nlong) chunk_base[jj] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  for (uint32_t b = threadIdx.x; b <= nb; b += 1024) {  // lower_bound(head, b * batch_items)
    const uint64_t key = (uint64_t)b * batch_items;
    uint32_t lo = 0, hi = nlong;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (head[mid] < key) lo = mid + 1; else hi = mid;
    }
    first[b] = lo;
  }
}

// ----------------------------------------------------------- dispatchers
// score_kernel<KIND> is shared by every (dim, k): its dynamic-smem attribute
// only grows; occupancy is cached per smem size.  (Host-side, per process.)
size_t g_score_attr[kMaxDevices][4];
size_t g_score_occ_smem[kMaxDevices][4];
int g_score_occ[kMaxDevices][4];

void sort_items(const BatchArgs& a, uint64_t items, const uint32_t* keys, const uint32_t* vals,
                int key_bits, cudaStream_t st, uint32_t* okeys = nullptr, uint32_t* ovals = nullptr) {
  size_t bytes = a.sort_temp_bytes;
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(a.sort_temp, bytes, keys, okeys ? okeys : a.skeys, vals,
                                           ovals ? ovals : a.svals, (int64_t)items, 0, key_bits, st));
}

// vector-lane pass 1 when the dimension fits one (NV = 1) or two (NV = 2)
// 16-byte vectors per lane; 0 = use the 8-lane-group kernel
template <int KIND>
int vec_width(uint32_t d) {
  if (KIND == 2) {
    const uint32_t h = d / 2;
    if (h % 2) return 0;
    return h <= 64 ? 1 : (h <= 128 ? 2 : 0);
  }
  if (d % 4) return 0;
  return d <= 128 ? 1 : (d <= 256 ? 2 : 0);
}

template <int KIND, int NV, bool REL, bool SH, bool GRAD>
void launch_vec_pass1_(const BatchArgs& a, uint64_t items, unsigned grid, cudaStream_t st) {
  const size_t smem = (size_t)(kSegThreads / 32) * kSegDepth * 2 * ((a.dim + 3) & ~3u) * 4;
  static size_t attr[kMaxDevices];  // per instantiation and device: grows only
  const int dev = current_device();
  if (smem > attr[dev]) {
    LGD_CUDA(cudaFuncSetAttribute(segment_pass1_vec<KIND, NV, REL, SH, GRAD>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[dev] = smem;
  }
  segment_pass1_vec<KIND, NV, REL, SH, GRAD><<<grid, kSegThreads, smem, st>>>(
      a, items, a.skeys, a.svals, a.span_list, a.span_count);
}
template <int KIND, int NV, bool REL, bool SH = false>
void launch_vec_pass1(const BatchArgs& a, uint64_t items, unsigned grid, cudaStream_t st) {
  if (REL ? a.grad_rels : a.grad_nodes)
    launch_vec_pass1_<KIND, NV, REL, SH, true>(a, items, grid, st);
  else
    launch_vec_pass1_<KIND, NV, REL, SH, false>(a, items, grid, st);
}

template <int KIND, int NV, bool SH, bool IR1, bool R64>
void launch_segment_heads_(const BatchArgs& a, uint64_t b0, uint64_t b1, cudaStream_t st) {
  const size_t smem =
      (size_t)(kSegThreads / 32) * seg_heads_depth<KIND>() * seg_slot_bytes((a.dim + 3) & ~3u) +
      ((K4_BULK_ALL || KIND == 3) ? (size_t)(kSegThreads / 32) * seg_heads_depth<KIND>() * 8 : 0);  // slot mbarriers
  static size_t attr[kMaxDevices];
  const int dev = current_device();
  if (smem > attr[dev]) {
    LGD_CUDA(cudaFuncSetAttribute(segment_heads<KIND, NV, SH, IR1, R64>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[dev] = smem;
  }
  // long segments first, on the side stream (disjoint rows), when there is one
  const LongList ll{a.long_head, a.long_end, a.long_chunk_base, a.long_first};
  cudaStream_t ls = st;
  if (a.side) {
    LGD_CUDA(cudaEventRecord(a.ev_long, st));
    LGD_CUDA(cudaStreamWaitEvent(a.side, a.ev_long, 0));
    ls = a.side;
  }
  long_chunks<KIND, NV, SH, IR1, R64><<<(unsigned)a.sm_count * 2, kSegThreads, 0, ls>>>(
      a, a.seg_keys, a.seg_vals, ll, a.seg_batch, a.part_first);
  LGD_LAUNCH_CHECK();
  long_combine<KIND, NV><<<(unsigned)a.sm_count, kSegThreads, 0, ls>>>(a, a.seg_keys, ll,
                                                                      a.seg_batch, a.part_first);
  LGD_LAUNCH_CHECK();
  if (a.side) LGD_CUDA(cudaEventRecord(a.ev_long_done, a.side));
  if (a.k4_ws == 2 && NV == 1) {  // K4 v4: flattened vectors
    const unsigned grid = (unsigned)ceil_div(ceil_div(b1 - b0, 32), kSegThreads / 32);
    segment_flat<KIND, SH, IR1, R64><<<grid, kSegThreads, 0, st>>>(a, a.seg_keys, a.seg_vals, b0,
                                                                   b1);
  } else if (a.k4_ws == 1) {
    const size_t wsm = ws_bar_bytes() + (size_t)kWsConsumers * kWsDepth * ws_slot_bytes((a.dim + 3) & ~3u);
    static size_t wattr[kMaxDevices];
    if (wsm > wattr[dev]) {
      LGD_CUDA(cudaFuncSetAttribute(segment_ws<KIND, NV, SH, IR1, R64>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm));
      wattr[dev] = wsm;
    }
    const unsigned wgrid = (unsigned)ceil_div(b1 - b0, (uint64_t)kWsChunks * 32);
    segment_ws<KIND, NV, SH, IR1, R64><<<wgrid, kWsThreads, wsm, st>>>(a, a.seg_keys, a.seg_vals,
                                                                       b0, b1);
  } else {
    const unsigned grid = (unsigned)ceil_div(ceil_div(b1 - b0, 32), kSegThreads / 32);
    segment_heads<KIND, NV, SH, IR1, R64><<<grid, kSegThreads, smem, st>>>(a, a.seg_keys,
                                                                           a.seg_vals, b0, b1);
  }
  LGD_LAUNCH_CHECK();
  if (a.side) LGD_CUDA(cudaStreamWaitEvent(st, a.ev_long_done, 0));
}

// K4 v2 for the node pass when the dimension has vector lanes.  The bucket's
// long-segment list (presorted) or a one-batch list built here for this
// batch's own sort.  ComplEx / TransE read K3's IR1 rows when the context
// keeps them (a.ir1), else recombine the snapshot with the relation row
// (same bits).
template <int KIND, bool SH>
bool segment_rows_node_pass(BatchArgs& a, uint64_t items, cudaStream_t st) {
  if (!a.seg_mode || a.grad_nodes) return false;
  const int nv = vec_width<KIND>(a.dim);
  if (nv == 0 || (KIND == 3 && SH)) return false;
  uint64_t b0 = a.seg_b0;
  if (a.seg_mode == 2) {  // this batch's sort: a one-batch list
    a.seg_keys = a.skeys;
    a.seg_vals = a.svals;
    a.seg_batch = 0;
    b0 = 0;
    launch_long_list(a.skeys, items, items, 1, a.seg_lists, st);
  }
  if constexpr (KIND != 3 || !SH) {
    constexpr bool kIr1 = k4_ir1(KIND) && !SH;
    constexpr bool kR64 = KIND != 0;
    const bool ir1 = kIr1 && a.ir1 != nullptr;
    const bool r64 = kR64 && a.rel64 != nullptr;
    auto go = [&](auto nvc, auto ir1c, auto r64c) {
      launch_segment_heads_<KIND, decltype(nvc)::value, SH, decltype(ir1c)::value,
                            decltype(r64c)::value>(a, b0, b0 + items, st);
    };
    using T = std::true_type;
    using F = std::false_type;
    using N1 = std::integral_constant<int, 1>;
    using N2 = std::integral_constant<int, 2>;
    if (nv == 1) {
      if (ir1) {
        if (r64) go(N1{}, std::integral_constant<bool, kIr1>{}, std::integral_constant<bool, kR64>{});
        else go(N1{}, std::integral_constant<bool, kIr1>{}, F{});
      } else {
        if (r64) go(N1{}, F{}, std::integral_constant<bool, kR64>{});
        else go(N1{}, F{}, F{});
      }
    } else {
      if (ir1) go(N2{}, std::integral_constant<bool, kIr1>{}, F{});
      else go(N2{}, F{}, F{});
    }
    (void)sizeof(T);
  }
  return true;
}

// shared-negative mode: node items are dst / shared negative / src (slots 0-2)
template <int KIND>
void run_segments_shared(const BatchArgs& a_in, uint64_t items, cudaStream_t st) {
  BatchArgs a = a_in;
  if (segment_rows_node_pass<KIND, true>(a, items, st)) return;
  LGD_CUDA(cudaMemsetAsync(a.span_count, 0, sizeof(unsigned int), st));
  const unsigned grid = ceil_div(ceil_div(items, 32), kSegThreads / 32);
  const int nv = vec_width<KIND>(a.dim);
  if (nv == 1) {
    launch_vec_pass1<KIND, 1, false, true>(a, items, grid, st);
  } else if (nv == 2) {
    launch_vec_pass1<KIND, 2, false, true>(a, items, grid, st);
  } else {
    throw std::invalid_argument("shared negatives need a vector-lane dimension");
  }
  LGD_LAUNCH_CHECK();
  segment_pass2<false><<<(unsigned)a.sm_count * 4, kPass2Threads, 0, st>>>(
      a, items, a.skeys, a.span_list, a.span_count);
  LGD_LAUNCH_CHECK();
}

template <int KIND, int NC>
void run_segments(const BatchArgs& a, uint64_t items, bool rel, cudaStream_t st) {
  LGD_CUDA(cudaMemsetAsync(a.span_count, 0, sizeof(unsigned int), st));
  const unsigned grid = ceil_div(ceil_div(items, 32), kSegThreads / 32);
  const unsigned grid2 = (unsigned)a.sm_count * 4;
  const int nv = vec_width<KIND>(a.dim);
  if (nv) {
    if (rel) {
      nv == 1 ? launch_vec_pass1<KIND, 1, true>(a, items, grid, st)
              : launch_vec_pass1<KIND, 2, true>(a, items, grid, st);
    } else {
      nv == 1 ? launch_vec_pass1<KIND, 1, false>(a, items, grid, st)
              : launch_vec_pass1<KIND, 2, false>(a, items, grid, st);
    }
    LGD_LAUNCH_CHECK();
    if (rel) {
      segment_pass2<true><<<grid2, kPass2Threads, 0, st>>>(a, items, a.skeys, a.span_list,
                                                            a.span_count);
    } else {
      segment_pass2<false><<<grid2, kPass2Threads, 0, st>>>(a, items, a.skeys, a.span_list,
                                                             a.span_count);
    }
    LGD_LAUNCH_CHECK();
    return;
  }
  if (rel) {
    segment_pass1<KIND, NC, true><<<grid, kSegThreads, 0, st>>>(a, items, a.skeys, a.svals,
                                                                a.span_list, a.span_count);
    LGD_LAUNCH_CHECK();
    segment_pass2<true><<<grid2, kPass2Threads, 0, st>>>(a, items, a.skeys, a.span_list,
                                                          a.span_count);
  } else {
    segment_pass1<KIND, NC, false><<<grid, kSegThreads, 0, st>>>(a, items, a.skeys, a.svals,
                                                                 a.span_list, a.span_count);
    LGD_LAUNCH_CHECK();
    segment_pass2<false><<<grid2, kPass2Threads, 0, st>>>(a, items, a.skeys, a.span_list,
                                                           a.span_count);
  }
  LGD_LAUNCH_CHECK();
}

__global__ void rel_apply_dense_kernel(const double* __restrict__ grad,
                                       const uint8_t* __restrict__ touched, float* __restrict__ th,
                                       float* __restrict__ st, uint64_t R, uint32_t d, double lr,
                                       double eps) {
  const uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= R || !touched[r]) return;
  for (uint32_t i = lane; i < d; i += 32) {
    float tv = th[r * d + i], sv = st[r * d + i];
    adagrad_fast(grad[r * d + i], tv, sv, lr, eps);
    th[r * d + i] = tv;
    st[r * d + i] = sv;
  }
}

// Relation pass, part 1: sort + segmented sums.  With a side stream it
// starts as soon as K3 is done and overlaps the node pass, writing dense
// gradients; rel_pass_finish then applies them after K4.
template <int KIND, int NC>
void rel_pass_start(const BatchArgs& a, cudaStream_t st) {
  if (KIND == 0) return;
  if (!a.side) {
    sort_items(a, a.P, a.rel_keys, a.iota, a.rel_key_bits, st);
    run_segments<KIND, NC>(a, a.P, true, st);
    return;
  }
  LGD_CUDA(cudaEventRecord(a.ev_scored, st));
  LGD_CUDA(cudaStreamWaitEvent(a.side, a.ev_scored, 0));
  // the batch loss is off the critical path too (K4 does not need it; the
  // next batch's K3 waits for ev_rel before it rewrites the per-positive losses)
  loss_reduce_kernel<<<1, 1024, 0, a.side>>>(a.loss, a.P, a.batch_loss_out, a.loss_parts);
  LGD_LAUNCH_CHECK();
  BatchArgs r = a;
  r.skeys = a.rel_skeys;
  r.svals = a.rel_svals;
  r.sort_temp = a.rel_sort_temp;
  r.sort_temp_bytes = a.rel_sort_temp_bytes;
  r.part_first = a.rel_part_first;
  r.part_last = a.rel_part_last;
  r.chunk_flags = a.rel_chunk_flags;
  r.span_list = a.rel_span_list;
  r.span_count = a.rel_span_count;
  r.grad_rels = a.rel_grad;
  r.grad_rel_flag = a.rel_touched;
  LGD_CUDA(cudaMemsetAsync(a.rel_touched, 0, a.num_rels, a.side));
  sort_items(r, a.P, a.rel_keys, a.iota, a.rel_key_bits, a.side);
  run_segments<KIND, NC>(r, a.P, true, a.side);
  LGD_CUDA(cudaEventRecord(a.ev_rel, a.side));
}
template <int KIND>
void rel_pass_finish(const BatchArgs& a, cudaStream_t st) {
  if (KIND == 0 || !a.side) return;
  LGD_CUDA(cudaStreamWaitEvent(st, a.ev_rel, 0));
  rel_apply_dense_kernel<<<ceil_div(a.num_rels * 32, 256), 256, 0, st>>>(
      a.rel_grad, a.rel_touched, a.rel_theta, a.rel_state, a.num_rels, a.dim, a.lr, a.eps);
  LGD_LAUNCH_CHECK();
}

// ------------------------------------- compact batch_gradients (operator)
// batch_gradients (train.cpp:280-340) as a GradientSet: the sorted unique
// node / relation ids and one FP64 gradient row each, O(unique rows) memory.
// Phase 1: the sorted contributions' segment heads (nodes and relations);
// phase 2: one warp per segment sums its contributions sequentially in the
// reference's order and writes row s of the output.
// segment heads of sorted keys: the first item, or a key change
struct HeadFlag {
  const uint32_t* keys;
  __host__ __device__ __forceinline__ bool operator()(const uint32_t& i) const {
    return i == 0 || keys[i] != keys[i - 1];
  }
};

void grads_phase1(const BatchArgs& a, uint64_t n, cudaStream_t st) {
  size_t bytes = a.gc->temp_bytes;
  LGD_CUDA(cub::DeviceSelect::If(a.gc->temp, bytes, thrust::counting_iterator<uint32_t>(0),
                                 a.gc->node_seg, a.gc->counts, (int64_t)n, HeadFlag{a.skeys}, st));
  if (a.gc->rel_seg) {
    sort_items(a, a.P, a.rel_keys, a.iota, a.rel_key_bits, st, a.gc->rel_skeys, a.gc->rel_svals);
    bytes = a.gc->temp_bytes;
    LGD_CUDA(cub::DeviceSelect::If(a.gc->temp, bytes, thrust::counting_iterator<uint32_t>(0),
                                   a.gc->rel_seg, a.gc->counts + 1, (int64_t)a.P,
                                   HeadFlag{a.gc->rel_skeys}, st));
  }
}

template <int KIND, int NV, bool REL>
__global__ void __launch_bounds__(kSegThreads) grad_segments(BatchArgs a, const uint32_t* __restrict__ skeys,
                                                             const uint32_t* __restrict__ svals, uint64_t n,
                                                             const uint32_t* __restrict__ seg, uint64_t nseg,
                                                             uint32_t* __restrict__ ids, double* __restrict__ out) {
  constexpr int NE = 4 * NV;
  const int lane = threadIdx.x & 31;
  const Lanes<KIND, NV> L(lane, a.dim);
  const SegCtx x{a.snap, a.mix, a.ir1, a.w, a.rel_theta, a.rel_keys, a.dim, a.k,
                 (uint32_t)a.slot_bits, (1u << a.slot_bits) - 1u,
                 (uint32_t)(a.slot_bits + a.rel_bits), a.rel_bits ? (1u << a.rel_bits) - 1u : 0u,
                 a.P * a.k, a.sh_G, nullptr};
  const uint64_t d = a.dim;
  const uint64_t nw = (uint64_t)gridDim.x * (kSegThreads / 32);
  for (uint64_t s = ((uint64_t)blockIdx.x * kSegThreads + threadIdx.x) >> 5; s < nseg; s += nw) {
    const uint32_t q0 = seg[s], q1 = s + 1 < nseg ? seg[s + 1] : (uint32_t)n;
    const uint32_t key = skeys[q0];
    const uint32_t row = REL ? key : from_pool(a, key);
    float own[NE];
    if (KIND == 3 && !REL) L.template ldf<true>(a.theta + (uint64_t)row * d, true, own);
    double acc[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) acc[e] = 0.0;
    for (uint32_t q = q0; q < q1; ++q) {  // every contribution, in order
      ItemRegs<NE> it;
      load_item<KIND, NV, REL, false>(x, L, __ldg(svals + q), true, it);
      add_loaded<KIND, NV, REL, false>(x, L, it, x.k, acc, own);
    }
    L.std_(out + s * d, acc);
    if (lane == 0) ids[s] = row;
  }
}

template <int KIND>
void grads_phase2_kind(const BatchArgs& a, uint64_t nn, uint64_t nr, uint32_t* node_ids,
                       double* node_grads, uint32_t* rel_ids, double* rel_grads, cudaStream_t st) {
  const int nv = vec_width<KIND>(a.dim);
  const unsigned grid = (unsigned)a.sm_count * 8;
  const uint64_t n = a.P * (a.k + 2);
  if (nn) {
    if (nv == 1)
      grad_segments<KIND, 1, false><<<grid, kSegThreads, 0, st>>>(a, a.skeys, a.svals, n, a.gc->node_seg, nn, node_ids, node_grads);
    else
      grad_segments<KIND, 2, false><<<grid, kSegThreads, 0, st>>>(a, a.skeys, a.svals, n, a.gc->node_seg, nn, node_ids, node_grads);
    LGD_LAUNCH_CHECK();
  }
  if (KIND != 0 && nr) {
    if (nv == 1)
      grad_segments<KIND, 1, true><<<grid, kSegThreads, 0, st>>>(a, a.gc->rel_skeys, a.gc->rel_svals, a.P, a.gc->rel_seg, nr, rel_ids, rel_grads);
    else
      grad_segments<KIND, 2, true><<<grid, kSegThreads, 0, st>>>(a, a.gc->rel_skeys, a.gc->rel_svals, a.P, a.gc->rel_seg, nr, rel_ids, rel_grads);
    LGD_LAUNCH_CHECK();
  }
}

template <int KIND, int NC>
void run_batch(const BatchArgs& a_in, cudaStream_t st, const BatchEvents* ev) {
  BatchArgs a = a_in;
  a.loss_parts = (KIND == 1 || KIND == 2) && a.side ? 1 : 0;
  auto rec = [&](int i) {
    if (ev && ev->enabled) LGD_CUDA(cudaEventRecord(ev->ev[i], st));
  };
  const uint32_t d = a.dim, k = a.k;
  const uint64_t P = a.P;
  const ScoreSmem L(d, k);
  constexpr int kW = score_warps<KIND>();
  const size_t smem = L.block_bytes(kW);
  const int tma = ((d % 4) == 0 && L.nrows <= 32) ? 1 : 0;
  rec(0);
  {
    // the dynamic-smem attribute only ever grows (it is shared by every
    // dimension / k this kernel serves); occupancy is cached per smem size
    const int dev = current_device();
    size_t* attr_set = g_score_attr[dev];
    size_t* occ_smem = g_score_occ_smem[dev];
    int* occ_val = g_score_occ[dev];
    if (smem > attr_set[KIND]) {
      LGD_CUDA(cudaFuncSetAttribute(score_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      attr_set[KIND] = smem;
    }
    if (occ_smem[KIND] != smem) {
      LGD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_val[KIND], score_kernel<KIND>,
                                                             kW * 32, smem));
      occ_smem[KIND] = smem;
    }
    const int per_sm = occ_val[KIND];
    if (per_sm < 1) throw std::invalid_argument("batch shape exceeds shared memory (k, dim)");
    const uint64_t blocks_needed = (P + kW - 1) / kW;
    const uint64_t cap = (uint64_t)per_sm * a.sm_count;
    const unsigned grid = (unsigned)(blocks_needed < cap ? blocks_needed : cap);
    score_kernel<KIND><<<grid, kW * 32, smem, st>>>(a, tma);
    LGD_LAUNCH_CHECK();
  }
  if (KIND == 0 && a.side) {  // Dot: the batch loss on the side stream, off K4's path
    LGD_CUDA(cudaEventRecord(a.ev_scored, st));
    LGD_CUDA(cudaStreamWaitEvent(a.side, a.ev_scored, 0));
    loss_reduce_kernel<<<1, 1024, 0, a.side>>>(a.loss, P, a.batch_loss_out, a.loss_parts);
    LGD_LAUNCH_CHECK();
    LGD_CUDA(cudaEventRecord(a.ev_rel, a.side));
  } else if (!(KIND != 0 && a.side)) {
    loss_reduce_kernel<<<1, 1024, 0, st>>>(a.loss, P, a.batch_loss_out, a.loss_parts);
    LGD_LAUNCH_CHECK();
  }
  rec(1);
  if (a.side) rel_pass_start<KIND, NC>(a, st);
  if (!a.presorted) sort_items(a, P * (k + 2), a.node_keys, a.node_vals, a.node_key_bits, st);
  if (a.gc) {  // compact gradients (batch_gradients): sorted runs + segment heads, no update
    grads_phase1(a, P * (k + 2), st);
    return;
  }
  rec(2);
  if (a.grad_nodes || !segment_rows_node_pass<KIND, false>(a, P * (k + 2), st))
    run_segments<KIND, NC>(a, P * (k + 2), false, st);
  rec(3);
  if (KIND == 0 && a.side) {
    // the next batch's K3 rewrites the per-positive losses
    LGD_CUDA(cudaStreamWaitEvent(st, a.ev_rel, 0));
  } else if (a.side) {
    rel_pass_finish<KIND>(a, st);
  } else {
    rel_pass_start<KIND, NC>(a, st);
  }
  rec(4);
}

// Shared-negative chunks: shared.cu computes loss, mix and the negatives'
// gradient rows on the tensor cores; the node / relation updates are the
// same segmented reduction + Adagrad as the exact path.
template <int KIND, int NC>
void run_batch_shared(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev) {
  auto rec = [&](int i) {
    if (ev && ev->enabled) LGD_CUDA(cudaEventRecord(ev->ev[i], st));
  };
  const uint64_t P = a.P;
  rec(0);
  launch_shared_scores(a, st);
  if (!(KIND != 0 && a.side)) {
    loss_reduce_kernel<<<1, 1024, 0, st>>>(a.loss, P, a.batch_loss_out, a.loss_parts);
    LGD_LAUNCH_CHECK();
  }
  rec(1);
  if (a.side) rel_pass_start<KIND, NC>(a, st);
  BatchArgs b = a;  // node items: (index << 2) | slot, slot 0 dst, 1 negative, 2 src
  b.k = 1;
  b.slot_bits = 2;
  b.rel_bits = 0;
  const uint64_t items = 2 * P + a.nch * a.k;
  sort_items(b, items, b.node_keys, b.node_vals, b.node_key_bits, st);
  rec(2);
  run_segments_shared<KIND>(b, items, st);
  rec(3);
  if (a.side) {
    rel_pass_finish<KIND>(a, st);
  } else {
    rel_pass_start<KIND, NC>(a, st);
  }
  rec(4);
}

template <int KIND>
void run_kind(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev) {
  const uint32_t lanes_elems = KIND == 2 ? a.dim / 2 : a.dim;
  const uint32_t nc = (lanes_elems + kGroup - 1) / kGroup;
  if constexpr (KIND == 3) {
    if (a.chunk) throw std::invalid_argument("shared negatives: TransE is not a dot-product score");
  } else if (a.chunk) {
    if (nc <= 4) return run_batch_shared<KIND, 4>(a, st, ev);
    if (nc <= 8) return run_batch_shared<KIND, 8>(a, st, ev);
    if (nc <= 16) return run_batch_shared<KIND, 16>(a, st, ev);
    return run_batch_shared<KIND, 32>(a, st, ev);
  }
  if (nc <= 1) return run_batch<KIND, 1>(a, st, ev);
  if (nc <= 2) return run_batch<KIND, 2>(a, st, ev);
  if (nc <= 4) return run_batch<KIND, 4>(a, st, ev);
  if (nc <= 8) return run_batch<KIND, 8>(a, st, ev);
  if (nc <= 13) return run_batch<KIND, 13>(a, st, ev);
  if (nc <= 16) return run_batch<KIND, 16>(a, st, ev);
  if (nc <= 32) return run_batch<KIND, 32>(a, st, ev);
  throw std::invalid_argument("embedding dimension too large (max 256, ComplEx 512)");
}

__global__ void rel_pack_kernel(const double* __restrict__ grad, const uint8_t* __restrict__ flag,
                                uint64_t R, uint32_t d, double* __restrict__ out) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R * (d + 1)) return;
  const uint64_t r = t / (d + 1), i = t - r * (d + 1);
  out[t] = i < d ? grad[r * d + i] : (flag[r] ? 1.0 : 0.0);
}

__global__ void rel_apply_kernel(const double* __restrict__ summed, float* __restrict__ th,
                                 float* __restrict__ st, uint64_t R, uint32_t d, double lr,
                                 double eps) {
  const uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= R || summed[r * (d + 1) + d] <= 0.0) return;  // row untouched by every rank
  for (uint32_t i = lane; i < d; i += 32) {
    float tv = th[r * d + i], sv = st[r * d + i];
    adagrad_fast(summed[r * (d + 1) + i], tv, sv, lr, eps);
    th[r * d + i] = tv;
    st[r * d + i] = sv;
  }
}

}  // namespace

void launch_rel_pack(const double* grad, const uint8_t* flag, uint64_t R, uint32_t d, double* out,
                     cudaStream_t st) {
  if (!R) return;
  rel_pack_kernel<<<ceil_div(R * (d + 1), 256), 256, 0, st>>>(grad, flag, R, d, out);
  LGD_LAUNCH_CHECK();
}

void launch_rel_apply(const double* summed, float* rel_theta, float* rel_state, uint64_t R,
                      uint32_t d, double lr, double eps, cudaStream_t st) {
  if (!R) return;
  rel_apply_kernel<<<ceil_div(R * 32, 256), 256, 0, st>>>(summed, rel_theta, rel_state, R, d, lr,
                                                           eps);
  LGD_LAUNCH_CHECK();
}

size_t batch_sort_temp_bytes(uint64_t max_items) {
  size_t bytes = 0;
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                           (uint32_t*)nullptr, (int64_t)(max_items ? max_items : 1),
                                           0, 32));
  return bytes;
}

// Bucket-level contribution keys, item i = e (k + 2) + s of the bucket's
// shuffled edge e (batch b = e / B, positive p = e - b B): s = 0 dst, 1..k
// negative s - 1, k + 1 src -- K3's per-batch layout (kb + slot), so a stable
// sort of (b, pool index) reproduces every batch's own sort.
__global__ void presort_keys_kernel(BatchArgs a, uint64_t m, uint64_t B, uint32_t* __restrict__ keys,
                                   uint32_t* __restrict__ vals) {
  const uint32_t k = a.k, k2 = k + 2;
  const uint64_t n = m * k2;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = i / k2;
    const uint32_t s = (uint32_t)(i - e * k2);
    const uint64_t b = e / B;
    const uint32_t p = (uint32_t)(e - b * B);
    const uint32_t id = s == 0 ? __ldg(a.edges + 3 * e + 2)
                        : s == k + 1 ? __ldg(a.edges + 3 * e)
                                     : __ldg(a.negs + e * k + (s - 1));
    const uint32_t rel = a.rel_bits ? __ldg(a.edges + 3 * e + 1) << a.slot_bits : 0u;
    keys[i] = ((uint32_t)b << a.node_key_bits) | to_pool(a, id);
    vals[i] = ((uint32_t)p << (a.slot_bits + a.rel_bits)) | rel | s;
  }
}

void launch_bucket_keys(const BatchArgs& a, uint64_t m, uint64_t B, uint32_t* keys,
                        uint32_t* vals, cudaStream_t st) {
  const uint64_t n = m * (a.k + 2);
  if (!n) return;
  const uint64_t blocks = ceil_div(n, 256);
  const unsigned grid = (unsigned)(blocks < (uint64_t)a.sm_count * 16 ? blocks : (uint64_t)a.sm_count * 16);
  presort_keys_kernel<<<grid, 256, 0, st>>>(a, m, B, keys, vals);
  LGD_LAUNCH_CHECK();
}

void launch_grads_phase2(const BatchArgs& a, uint64_t nn, uint64_t nr, uint32_t* node_ids,
                         double* node_grads, uint32_t* rel_ids, double* rel_grads, cudaStream_t st) {
  switch (a.kind) {
    case 0: return grads_phase2_kind<0>(a, nn, nr, node_ids, node_grads, rel_ids, rel_grads, st);
    case 1: return grads_phase2_kind<1>(a, nn, nr, node_ids, node_grads, rel_ids, rel_grads, st);
    case 2: return grads_phase2_kind<2>(a, nn, nr, node_ids, node_grads, rel_ids, rel_grads, st);
    default: return grads_phase2_kind<3>(a, nn, nr, node_ids, node_grads, rel_ids, rel_grads, st);
  }
}

size_t grads_select_temp_bytes(uint64_t max_items) {
  size_t b = 0;
  LGD_CUDA(cub::DeviceSelect::If(nullptr, b, thrust::counting_iterator<uint32_t>(0),
                                 (uint32_t*)nullptr, (uint32_t*)nullptr,
                                 (int64_t)(max_items ? max_items : 1), HeadFlag{nullptr}));
  return b;
}

int k4_vec_width(int kind, uint32_t dim) {
  switch (kind) {
    case 0: return vec_width<0>(dim);
    case 1: return vec_width<1>(dim);
    case 2: return vec_width<2>(dim);
    default: return vec_width<3>(dim);
  }
}

size_t long_list_temp_bytes(uint64_t max_items) {
  size_t b = 0;
  LGD_CUDA(cub::DeviceSelect::If(nullptr, b, thrust::counting_iterator<uint32_t>(0),
                                 (uint32_t*)nullptr, (uint32_t*)nullptr,
                                 (int64_t)(max_items ? max_items : 1), LongHead{nullptr, 0}));
  return b;
}

void launch_long_list(const uint32_t* keys, uint64_t n, uint64_t batch_items, uint32_t nb,
                      const SegLists& L, cudaStream_t st) {
  if (!n) return;
  size_t bytes = L.temp_bytes;  // heads of segments longer than kLongSeg, ascending
  LGD_CUDA(cub::DeviceSelect::If(L.temp, bytes, thrust::counting_iterator<uint32_t>(0),
                                 L.long_head, L.nlong, (int64_t)n, LongHead{keys, n}, st));
  long_index_kernel<<<1, 1024, 0, st>>>(keys, n, L.long_head, L.nlong, batch_items, nb, L.long_end,
                                        L.long_chunk_base, L.long_first);
  LGD_LAUNCH_CHECK();
}

size_t bucket_sort_temp_bytes(uint64_t max_items) {
  size_t bytes = 0;
  cub::DoubleBuffer<uint32_t> k(nullptr, nullptr), v(nullptr, nullptr);
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v,
                                           (int64_t)(max_items ? max_items : 1), 0, 32));
  return bytes;
}

int sort_bucket(void* temp, size_t temp_bytes, uint32_t* keys[2], uint32_t* vals[2],
                uint64_t items, int key_bits, cudaStream_t st) {
  cub::DoubleBuffer<uint32_t> k(keys[0], keys[1]), v(vals[0], vals[1]);
  size_t bytes = temp_bytes;
  LGD_CUDA(cub::DeviceRadixSort::SortPairs(temp, bytes, k, v, (int64_t)items, 0, key_bits, st));
  return k.selector;
}

size_t score_smem_bytes(uint32_t dim, uint32_t k) {
  return ScoreSmem(dim, k).block_bytes(kScoreWarps);  // the largest block of any model
}

#ifdef LGD_TRACE
extern "C" int lgd_debug_trace_k4(unsigned long long* out) {
  unsigned int z[8] = {0};
  cudaMemcpyFromSymbol(out, g_trace_k4, sizeof(g_trace_k4));
  return cudaMemcpyToSymbol(g_trace_k4_n, z, sizeof z) == cudaSuccess ? 0 : 4;
}
#endif

void launch_train_batch(const BatchArgs& a, cudaStream_t st, const BatchEvents* ev) {
  if (a.P == 0) return;
  switch (a.kind) {
    case 0:
      return run_kind<0>(a, st, ev);
    case 1:
      return run_kind<1>(a, st, ev);
    case 2:
      return run_kind<2>(a, st, ev);
    default:
      return run_kind<3>(a, st, ev);
  }
}

}  // namespace lgd
