// evaluate.cu -- K6: evaluate() (train.cpp:375-412) on the device.
//
// Test edges run in tiles (bounded candidate scratch):
//   candidates  one thread per test edge replays that edge's own stream
//               Rng(derive_seed(seed, "evay", t)) sequentially, so next_below
//               rejections are handled exactly as in the reference.
//   scores      one warp per test edge.  IR1 = combine_src_rel(src, rel) in
//               FP64 in shared memory; the true destination and the candidate
//               rows are staged 32 at a time into a per-warp shared-memory
//               double buffer by cp.async (coalesced 16-byte copies, the next
//               32 rows in flight while the current ones are scored), and lane
//               l scores row l SEQUENTIALLY over the dimension -- the
//               reference's own FP64 summation order (train.cpp:392-396), so a
//               near-tie lands on the same side of the pessimistic ">=" rule.
//               The staged row stride is padded to an odd number of 16-byte
//               units, so the lanes' float4 reads are bank-conflict free.
//   reduction   per-edge reciprocal ranks and hits go to the host, which sums
//               them in edge order (train.cpp:406-411), bit for bit.
// Bound: HBM -- (ncand + 2) rows of 4d bytes per test edge (~400 KB at TW's
// d = 100), gathered at random.
#include "common.cuh"
#include "evaluate.cuh"
#include "rng.cuh"

namespace lgd {

namespace {

constexpr int kEvalWarps = 4;
#ifndef EVAL_BULK  // candidate rows staged by one TMA bulk copy per row (0: 16-byte cp.async pieces)
#define EVAL_BULK 1
#endif

__device__ __forceinline__ void ev_bar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void ev_bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ev_bar_wait(uint32_t bar, uint32_t phase) {
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

__global__ void eval_candidates_kernel(uint64_t seed, uint64_t t0, uint64_t T, uint32_t ncand,
                                       uint64_t V, uint32_t* __restrict__ cand) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= T) return;
  Xo x = xo_seed(derive_seed(seed, kTagEval, t0 + i));
  const Below bd = make_below(V);
  for (uint32_t c = 0; c < ncand; ++c) {
    uint64_t r;
    do {
      r = xo_next(x);
    } while (r < bd.threshold);
    const uint64_t id = mod_below(r, bd);  // r % V by the precomputed reciprocal
    LGD_DCHECK(id == r % V, "candidate id", id);
    cand[i * ncand + c] = (uint32_t)id;
  }
}

// per warp: IR1 [dpad] f64, then two buffers of 32 rows; the row stride is an
// odd number of 16-byte units so lane l's float4 reads of row l hit distinct
// banks in every quarter warp
struct EvalSmem {
  uint32_t dpad, rstride;
  size_t ir1_off, rows_off, bars_off, warp_bytes;
  __host__ __device__ explicit EvalSmem(uint32_t d) {
    dpad = (d + 3) & ~3u;
    rstride = (dpad / 4) % 2 ? dpad : dpad + 4;
    ir1_off = 0;
    rows_off = (size_t)dpad * 8;
    bars_off = rows_off + 2 * 32 * (size_t)rstride * 4;
    warp_bytes = bars_off + 16;  // + one mbarrier per row buffer (bulk staging)
  }
};

template <int KIND>
__global__ void __launch_bounds__(kEvalWarps * 32) eval_score_kernel(
    uint32_t d, const float* __restrict__ theta, const float* __restrict__ rel,
    const uint32_t* __restrict__ edges, uint64_t T, uint32_t ncand,
    const uint32_t* __restrict__ cand, uint32_t hits_k, double* __restrict__ rr,
    double* __restrict__ hit) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const EvalSmem L(d);
  unsigned char* wb = smem + warp * L.warp_bytes;
  double* ir1 = reinterpret_cast<double*>(wb + L.ir1_off);
  float* rows = reinterpret_cast<float*>(wb + L.rows_off);
  const uint32_t rs = L.rstride, h = d / 2, nv = d / 4;
  const bool vec = (d & 3) == 0;
  const uint64_t nwarps = (uint64_t)gridDim.x * kEvalWarps;
  const uint32_t nrows = ncand + 1;  // row 0: the true destination
  const bool bulk = EVAL_BULK && vec;
  const uint32_t bars = (uint32_t)__cvta_generic_to_shared(wb + L.bars_off);
  if (bulk) {
    if (lane == 0) {
      ev_bar_init(bars);
      ev_bar_init(bars + 8);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  uint32_t gchunk = 0;  // chunks staged by this warp so far: buffer gchunk & 1, phase (gchunk >> 1) & 1
  for (uint64_t t = (uint64_t)blockIdx.x * kEvalWarps + warp; t < T; t += nwarps) {
    const uint32_t s = edges[3 * t], r = edges[3 * t + 1], dd = edges[3 * t + 2];
    const uint32_t* my = cand + t * ncand;
    LGD_DCHECK(t < T && (uint64_t)(my - cand) + ncand <= T * (uint64_t)ncand, "eval tile", t);
    // IR1 = combine_src_rel (train.cpp:39-60), per element as the reference
    const float* sr = theta + (size_t)s * d;
    const float* rl = KIND != 0 ? rel + (size_t)r * d : nullptr;
    for (uint32_t i = lane; i < d; i += 32) {
      double x;
      if (KIND == 0) {
        x = sr[i];
      } else if (KIND == 1) {
        x = (double)sr[i] * (double)rl[i];
      } else if (KIND == 3) {
        x = (double)sr[i] + (double)rl[i];
      } else {
        const uint32_t j = i < h ? i : i - h;
        const double a = sr[j], b = sr[j + h], p = rl[j], q = rl[j + h];
        x = i < h ? a * p - b * q : a * q + b * p;
      }
      ir1[i] = x;
    }
    auto row_id = [&](uint32_t q) { return q == 0 ? dd : my[q - 1]; };
    // stage rows [32 c, 32 c + 32) into buffer c & 1 (zero rows past the end)
    const uint32_t g0 = gchunk;  // this edge's chunk c is the warp's chunk g0 + c
    auto stage = [&](uint32_t c) {
      const uint32_t gb = (g0 + c) & 1;
      float* buf = rows + gb * 32 * rs;
      const uint32_t q0 = 32 * c;
      const uint32_t my_id = q0 + lane < nrows ? row_id(q0 + lane) : 0;
      if (bulk) {  // lane q copies row q: one bulk copy per row, counted on the buffer's mbarrier
        const uint32_t n = nrows - q0 < 32 ? nrows - q0 : 32;
        if (lane == 0) ev_bar_expect(bars + 8 * gb, n * d * 4);
        __syncwarp();
        if (lane < (int)n)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
              "[%3];" ::"r"((uint32_t)__cvta_generic_to_shared(buf + lane * rs)),
              "l"(theta + (size_t)my_id * d), "r"(d * 4), "r"(bars + 8 * gb)
              : "memory");
        return;
      }
      for (int q = 0; q < 32; ++q) {
        const uint32_t id = __shfl_sync(0xffffffffu, my_id, q);
        if (q0 + q >= nrows) break;
        const float* src = theta + (size_t)id * d;
        float* dst = buf + q * rs;
        if (vec) {
          for (uint32_t v = lane; v < nv; v += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst + 4 * v)),
                         "l"(src + 4 * v)
                         : "memory");
        } else {
          for (uint32_t i = lane; i < d; i += 32)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst + i)),
                         "l"(src + i)
                         : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const uint32_t nchunks = (nrows + 31) / 32;
    stage(0);
    double truth = 0.0;
    uint32_t beaten = 0;
    for (uint32_t c = 0; c < nchunks; ++c) {
      if (bulk) {
        if (c + 1 < nchunks) stage(c + 1);
        ev_bar_wait(bars + 8 * ((g0 + c) & 1), ((g0 + c) >> 1) & 1);
      } else if (c + 1 < nchunks) {
        stage(c + 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      const uint32_t q = 32 * c + lane;
      const float* row = rows + ((g0 + c) & 1) * 32 * rs + lane * rs;
      double f = 0.0;
      if (q < nrows) {
        if (KIND == 3) {  // -||u - t||, squares summed sequentially
          if (vec) {
            for (uint32_t i = 0; i < d; i += 4) {
              const float4 v = *reinterpret_cast<const float4*>(row + i);
              const double2 x0 = *reinterpret_cast<const double2*>(ir1 + i);
              const double2 x1 = *reinterpret_cast<const double2*>(ir1 + i + 2);
              const double z0 = x0.x - (double)v.x, z1 = x0.y - (double)v.y;
              const double z2 = x1.x - (double)v.z, z3 = x1.y - (double)v.w;
              f += z0 * z0;
              f += z1 * z1;
              f += z2 * z2;
              f += z3 * z3;
            }
          } else {
            for (uint32_t i = 0; i < d; ++i) {
              const double z = ir1[i] - (double)row[i];
              f += z * z;
            }
          }
          f = -sqrt(f);
        } else if (vec) {
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
      }
      if (c == 0) truth = __shfl_sync(0xffffffffu, f, 0);
      const bool b = q >= 1 && q < nrows && f >= truth;  // pessimistic ties (train.cpp:401-403)
      beaten += __popc(__ballot_sync(0xffffffffu, b));
      __syncwarp();  // the buffer is restaged by the next iteration's stage(c + 2)
    }
    gchunk = g0 + nchunks;
    if (lane == 0) {
      const uint64_t rank = 1ull + beaten;
      rr[t] = 1.0 / (double)rank;
      hit[t] = rank <= hits_k ? 1.0 : 0.0;
    }
    __syncwarp();  // ir1 is rewritten by the next test edge
  }
}

template <int KIND>
void launch_scores(const EvalArgs& a, uint64_t T, const uint32_t* edges, double* rr, double* hit,
                   cudaStream_t st) {
  const EvalSmem L(a.dim);
  const size_t smem = kEvalWarps * L.warp_bytes;
  static size_t attr[kMaxDevices];
  const int dev = current_device();
  if (smem > attr[dev]) {
    LGD_CUDA(cudaFuncSetAttribute(eval_score_kernel<KIND>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[dev] = smem;
  }
  int occ = 0;
  LGD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, eval_score_kernel<KIND>,
                                                         kEvalWarps * 32, smem));
  int sms = 148;
  LGD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const uint64_t blocks = std::min<uint64_t>(ceil_div(T, kEvalWarps), (uint64_t)std::max(occ, 1) * sms);
  eval_score_kernel<KIND><<<(unsigned)blocks, kEvalWarps * 32, smem, st>>>(
      a.dim, a.theta, a.rel, edges, T, a.ncand, a.cand, a.hits_k, rr, hit);
  LGD_LAUNCH_CHECK();
}

}  // namespace

size_t eval_smem_bytes(uint32_t dim) { return kEvalWarps * EvalSmem(dim).warp_bytes; }

void launch_evaluate_tile(const EvalArgs& a, uint64_t t0, uint64_t T, cudaStream_t st) {
  eval_candidates_kernel<<<ceil_div(T, 128), 128, 0, st>>>(a.seed, t0, T, a.ncand, a.V, a.cand);
  LGD_LAUNCH_CHECK();
  const uint32_t* edges = a.edges + 3 * t0;
  double* rr = a.rr + t0;
  double* hit = a.hit + t0;
  switch (a.kind) {
    case 0: launch_scores<0>(a, T, edges, rr, hit, st); break;
    case 1: launch_scores<1>(a, T, edges, rr, hit, st); break;
    case 2: launch_scores<2>(a, T, edges, rr, hit, st); break;
    default: launch_scores<3>(a, T, edges, rr, hit, st); break;
  }
}

}  // namespace lgd
