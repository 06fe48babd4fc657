// shared.cu -- shared-negative chunks on the 5th-generation tensor cores.
//
// Mode: every run of C consecutive
// positives of a batch (a "chunk") shares the same k negatives, drawn from the
// bucket stream right where the reference draws its P k per-positive ones
// (ceil(P / C) k draws per batch).  The reference math on the expanded
// negative list is the oracle; scores are a dense chunk x negatives x dim
// contraction, computed here with tcgen05.mma kind::tf32 (FP32 accumulate in
// TMEM), in two kernels that never materialise the P x k weight matrix:
//
//   SG2 mix     per 128-positive tile: S = IR1 N^T block by block with an
//               online softmax; the unnormalised weights into TMEM, acc += W N
//               on the tensor core  ->  mix = acc / Z - dst, the row's weight
//               offset c_p = M_p log2e + log2 Z_p and loss_p
//   SG3 grad    per (chunk, 128 negatives): S^T = N IR1^T recomputed per
//               128-positive slice, W^T = 2^(S^T log2e - c) into TMEM,
//               G += W^T IR1
// (round 2: a separate statistics pass, SG1, was folded into SG2)
//
// Operands live in global memory in the tcgen05 K-major "core matrix" layout
// without swizzle (8 rows x 16 bytes per 128-byte core matrix, the K-adjacent
// core matrices 128 bytes apart), so every tile is one contiguous TMA bulk
// copy:
//   byte(r, c) = ((r / 8) * (cols / 4) + c / 4) * 128 + (r % 8) * 16 + (c % 4) * 4
// kind::tf32 reads MN-major operands only through the 128B/32B-atom swizzle
// (a no-swizzle MN-major B reads as zeros -- profiles/micro/umma_probe.cu), so
// the second use of IR1 and of the negatives reads transposed K-major copies
// (IR1^T per 64-positive slice, N^T per 64-negative block) that the prep and
// gather kernels write next to the row-major ones.
// IR1 = combine_src_rel(s, r) (train.cpp:39-60) and the negative rows are
// rounded to TF32 (cvt.rna) when they are written.  The node-gradient
// contributions (dst: -IR1, negative: G row, src: adj(mix)) then go through
// the same sort-by-node segmented reduction and Adagrad as the exact path.
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "train.cuh"

namespace lgd {

namespace {

constexpr int kMixBlk = 128;   // negatives per S / mix block (SG2)
constexpr int kGradSlice = 128;  // positives per S^T / G slice (SG3)

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(b))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   saddr(dst_smem)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]^T, TF32 inputs, FP32 accumulate
__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive on the mbarrier once every previously issued MMA of this thread is done
__device__ __forceinline__ void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   saddr(b))
               : "memory");
}
// 16 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Shared-memory matrix descriptor, no swizzle: lbo = byte distance of the
// core matrices adjacent in the leading (K for K-major, MN otherwise... see
// the per-GEMM comments) dimension, sbo = the other one.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, layout SWIZZLE_NONE (0)
}
// Instruction descriptor: kind::tf32, FP32 accumulator, M x N, operand majors
__host__ __device__ constexpr uint32_t instr_desc(uint32_t M, uint32_t N, bool a_mn, bool b_mn) {
  return (1u << 4)                    // D format F32
         | (2u << 7) | (2u << 10)     // A, B format TF32
         | ((a_mn ? 1u : 0u) << 15)   // A major
         | ((b_mn ? 1u : 0u) << 16)   // B major
         | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ uint32_t pool_index(const BatchArgs& a, uint32_t id) {
  uint64_t prev = 0;
  for (int i = 0; i < a.pool_n; ++i) {
    const uint64_t cnt = a.pool_end[i] - prev;
    if (id >= a.pool_first[i] && id - a.pool_first[i] < cnt)
      return (uint32_t)(prev + id - a.pool_first[i]);
    prev = a.pool_end[i];
  }
  return 0xffffffffu;
}

// ------------------------------------------------------------ prep kernels
// Both run one block per 64 rows: every warp fills 8 rows of a shared-memory
// tile, then the block writes the tile in both core-matrix layouts (the
// K-major row block and its transpose) as consecutive 16-byte chunks.
constexpr int kPrepRows = 64;

__device__ __forceinline__ void write_core_layouts(const float* tile, uint32_t ts, uint32_t dp,
                                                   unsigned char* rows_out,
                                                   unsigned char* cols_out) {
  // rows_out: 64 rows x dp (cols = dp); cols_out: dp rows x 64 (cols = 64)
  const uint32_t chunks = 64 * dp / 4;  // 16-byte chunks per layout
  for (uint32_t i = threadIdx.x; i < chunks; i += blockDim.x) {
    {  // K-major over dp: chunk i = core matrix i / 8, row i % 8 of it
      const uint32_t cmi = i >> 3, rg = cmi / (dp / 4), qc = cmi - rg * (dp / 4);
      const uint32_t r = rg * 8 + (i & 7);
      *reinterpret_cast<float4*>(rows_out + 16ull * i) =
          *reinterpret_cast<const float4*>(tile + r * ts + 4 * qc);
    }
    {  // transpose: rows = dims, K = the 64 rows
      const uint32_t cmi = i >> 3, ig = cmi >> 4, qc = cmi & 15;
      const uint32_t e = ig * 8 + (i & 7);
      float4 v;
      v.x = tile[(4 * qc + 0) * ts + e];
      v.y = tile[(4 * qc + 1) * ts + e];
      v.z = tile[(4 * qc + 2) * ts + e];
      v.w = tile[(4 * qc + 3) * ts + e];
      *reinterpret_cast<float4*>(cols_out + 16ull * i) = v;
    }
  }
}

// IR1 (TF32) of 64 padded tile rows, the positive score in FP64, snap = the
// src row, the dst row (tile-major, for SG2's tail), the dst / src
// contribution items and the relation key.  Warp w
// fills rows 8w .. 8w + 7: their edges are fetched lane-parallel, then every
// row is read with 16-byte (ComplEx: 8-byte re / im pair) loads.
template <int KIND>
__global__ void __launch_bounds__(256) shared_prep_kernel(BatchArgs a) {
  extern __shared__ __align__(16) float ptile[];
  const uint32_t C = a.chunk, d = a.dim, dp = a.dpad, h = d / 2, ts = dp + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t rows_per_chunk = (uint64_t)a.tpc * 128;
  const uint64_t row0 = (uint64_t)blockIdx.x * kPrepRows;
  // lane i < 8: row 8 warp + i
  uint32_t es = 0, er = 0, et = 0;
  uint64_t ep = 0;
  bool ev = false;
  if (lane < 8) {
    const uint64_t row = row0 + warp * 8 + lane;
    const uint64_t c = row / rows_per_chunk, r = row - c * rows_per_chunk;
    ep = c * C + r;
    ev = r < C && ep < a.P;
    if (ev) {
      es = a.edges[3 * ep];
      er = a.edges[3 * ep + 1];
      et = a.edges[3 * ep + 2];
    }
  }
  const uint32_t vmask = __ballot_sync(0xffffffffu, ev);
#pragma unroll 2
  for (int i = 0; i < 8; ++i) {
    const int rr = warp * 8 + i;
    float* trow = ptile + rr * ts;
    if (!((vmask >> i) & 1u)) {
      for (uint32_t e = lane; e < dp; e += 32) trow[e] = 0.f;
      continue;
    }
    const uint32_t s = __shfl_sync(0xffffffffu, es, i);
    const uint32_t rel = __shfl_sync(0xffffffffu, er, i);
    const uint32_t t = __shfl_sync(0xffffffffu, et, i);
    const uint64_t p = __shfl_sync(0xffffffffu, ep, i);
    const float* srow = a.theta + (size_t)s * d;
    const float* rrow = KIND != 0 ? a.rel_theta + (size_t)rel * d : nullptr;
    const float* drow = a.theta + (size_t)t * d;
    double pos = 0.0;
    if (KIND == 2) {  // lane l: real indices 2l, 2l + 1 and their imaginary partners
      if (2 * (uint32_t)lane < h) {
        const uint32_t j = 2 * lane;
        const float2 sr = *reinterpret_cast<const float2*>(srow + j);
        const float2 si = *reinterpret_cast<const float2*>(srow + j + h);
        const float2 qr = *reinterpret_cast<const float2*>(rrow + j);
        const float2 qi = *reinterpret_cast<const float2*>(rrow + j + h);
        const float2 dr = *reinterpret_cast<const float2*>(drow + j);
        const float2 di = *reinterpret_cast<const float2*>(drow + j + h);
        const double xr0 = (double)sr.x * qr.x - (double)si.x * qi.x;
        const double xr1 = (double)sr.y * qr.y - (double)si.y * qi.y;
        const double xi0 = (double)sr.x * qi.x + (double)si.x * qr.x;
        const double xi1 = (double)sr.y * qi.y + (double)si.y * qr.y;
        pos = xr0 * dr.x + xr1 * dr.y + xi0 * di.x + xi1 * di.y;
        *reinterpret_cast<float2*>(a.snap + p * d + j) = sr;
        *reinterpret_cast<float2*>(a.snap + p * d + j + h) = si;
        *reinterpret_cast<float2*>(a.sh_D + (row0 + rr) * d + j) = dr;
        *reinterpret_cast<float2*>(a.sh_D + (row0 + rr) * d + j + h) = di;
        trow[j] = to_tf32((float)xr0);
        trow[j + 1] = to_tf32((float)xr1);
        trow[j + h] = to_tf32((float)xi0);
        trow[j + h + 1] = to_tf32((float)xi1);
      }
    } else if (4 * (uint32_t)lane < d) {  // lane l: elements 4l .. 4l + 3
      const uint32_t e = 4 * lane;
      const float4 sv = *reinterpret_cast<const float4*>(srow + e);
      const float4 dv = *reinterpret_cast<const float4*>(drow + e);
      float4 qv = make_float4(1.f, 1.f, 1.f, 1.f);
      if (KIND != 0) qv = *reinterpret_cast<const float4*>(rrow + e);
      const double x0 = KIND == 0 ? (double)sv.x : (double)sv.x * qv.x;
      const double x1 = KIND == 0 ? (double)sv.y : (double)sv.y * qv.y;
      const double x2 = KIND == 0 ? (double)sv.z : (double)sv.z * qv.z;
      const double x3 = KIND == 0 ? (double)sv.w : (double)sv.w * qv.w;
      pos = x0 * dv.x + x1 * dv.y + x2 * dv.z + x3 * dv.w;
      *reinterpret_cast<float4*>(a.snap + p * d + e) = sv;
      *reinterpret_cast<float4*>(a.sh_D + (row0 + rr) * d + e) = dv;
      *reinterpret_cast<float4*>(trow + e) =
          make_float4(to_tf32((float)x0), to_tf32((float)x1), to_tf32((float)x2),
                      to_tf32((float)x3));
    }
    for (uint32_t e = d + lane; e < dp; e += 32) trow[e] = 0.f;
#pragma unroll
    for (int off = 16; off; off >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, off);
    if (lane == 0) {
      a.sh_pos[p] = pos;
      a.node_keys[2 * p] = pool_index(a, t);
      a.node_vals[2 * p] = (uint32_t)(p << 2);  // slot 0: dst
      a.node_keys[2 * p + 1] = pool_index(a, s);
      a.node_vals[2 * p + 1] = (uint32_t)(p << 2) | 2u;  // slot 2: src
      if (KIND != 0) a.rel_keys[p] = rel;
    }
  }
  __syncthreads();
  write_core_layouts(ptile, ts, dp, reinterpret_cast<unsigned char*>(a.sh_A) + row0 * dp * 4,
                     reinterpret_cast<unsigned char*>(a.sh_AT) + row0 * dp * 4);
}

// TF32 rows of 64 padded negative slots (chunk, j < kpad) and, for j < k,
// the negatives' contribution items (16-byte loads, ids lane-parallel).
__global__ void __launch_bounds__(256) shared_gather_kernel(BatchArgs a) {
  extern __shared__ __align__(16) float ptile[];
  const uint32_t d = a.dim, dp = a.dpad, k = a.k, kp = a.kpad, ts = dp + 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t slot0 = (uint64_t)blockIdx.x * kPrepRows;
  uint32_t myid = 0;
  bool mv = false;
  uint64_t mc = 0;
  uint32_t mj = 0;
  if (lane < 8) {
    const uint64_t slot = slot0 + warp * 8 + lane;
    mc = slot / kp;
    mj = (uint32_t)(slot - mc * kp);
    mv = mj < k;
    if (mv) myid = a.negs[mc * k + mj];
  }
  const uint32_t vmask = __ballot_sync(0xffffffffu, mv);
  // the warp's rows by TMA bulk copies (lane i < 8 copies row i; random rows
  // gathered per lane are load-path bound), then TF32 rounding in place
  __shared__ uint64_t gbar[8];
  if (lane == 0) {
    bar_init(gbar + warp, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    bar_expect(gbar + warp, __popc(vmask) * d * 4);
  }
  __syncwarp();
  if (mv) bulk_load(ptile + (warp * 8 + lane) * ts, a.theta + (size_t)myid * d, d * 4, gbar + warp);
#pragma unroll 4
  for (int i = 0; i < 8; ++i) {  // zero the padded slots and the columns past d
    float* trow = ptile + (warp * 8 + i) * ts;
    for (uint32_t e = ((vmask >> i) & 1u ? d : 0u) + lane; e < dp; e += 32) trow[e] = 0.f;
  }
  bar_wait(gbar + warp, 0);
#pragma unroll 4
  for (int i = 0; i < 8; ++i) {
    if (!((vmask >> i) & 1u) || 4 * (uint32_t)lane >= d) continue;
    float4* t4 = reinterpret_cast<float4*>(ptile + (warp * 8 + i) * ts + 4 * lane);
    const float4 v = *t4;
    *t4 = make_float4(to_tf32(v.x), to_tf32(v.y), to_tf32(v.z), to_tf32(v.w));
  }
  if (lane < 8 && mv) {
    const uint64_t item = 2 * a.P + mc * k + mj;
    a.node_keys[item] = pool_index(a, myid);
    a.node_vals[item] = (uint32_t)((mc * kp + mj) << 2) | 1u;  // slot 1: shared negative
  }
  __syncthreads();
  write_core_layouts(ptile, ts, dp, reinterpret_cast<unsigned char*>(a.sh_B) + slot0 * dp * 4,
                     reinterpret_cast<unsigned char*>(a.sh_BT) + slot0 * dp * 4);
}

// --------------------------------------------------------- tensor-core GEMMs
struct TileGeom {  // a 128-positive tile of one chunk
  uint64_t c;        // chunk
  uint64_t row0;     // first tile row (global padded row index)
  uint32_t valid;    // valid rows in this tile
};
__device__ __forceinline__ TileGeom tile_geom(const BatchArgs& a, uint64_t t) {
  TileGeom g;
  g.c = t / a.tpc;
  const uint64_t in_chunk = (t - g.c * a.tpc) * 128;
  const uint64_t left = a.P - g.c * a.chunk;
  const uint64_t chunk_rows = left < a.chunk ? left : a.chunk;
  g.row0 = t * 128;
  const uint64_t rem = in_chunk < chunk_rows ? chunk_rows - in_chunk : 0;
  g.valid = (uint32_t)(rem < 128 ? rem : 128);
  return g;
}

// Pipelining (both kernels): warp specialised.  Warp 8 (lane 0) issues the
// S MMAs and their operands' bulk copies, warp 9 (lane 0) the W-operand MMAs
// (acc / G) and theirs -- two issuing threads, so the two MMA chains
// interleave on the tensor pipe instead of one queueing behind the other;
// warps 0-7 are the epilogue: warp w reads TMEM lane quarter w % 4 (its 32
// tile rows) and column half w / 4 of each 128-column block.  S lives in two
// TMEM buffers, so the MMA of block b + 1 runs while the epilogue drains
// block b.  mbarriers:
//   ld_*   bulk copy landed (complete_tx)       mma_s[2]  S MMA done (commit)
//   epi[2] the 8 epilogue warps read S buffer    wrdy      W written (8 warps)
//   mma_w  the W-operand MMA done (commit): W and that block's operand free
// Phase parity of a barrier used once per block b with buffer b % 2 is
// (b / 2) & 1; of one used once per block, b & 1.
constexpr int kWarps = 8;                      // epilogue warps
constexpr int kThreadsSG = (kWarps + 2) * 32;  // + the two issuing warps

// Developer timeline of one CTA (build with -DLGD_TRACE; not in the product .so)
#ifdef LGD_TRACE
// [kernel: SG1 (retired), SG2, SG3][control warp, epilogue warp 1][slot]
__device__ unsigned long long g_trace[3][2][4096];
#define SG_TRACE(kid, slot)                                                            \
  do {                                                                                 \
    if (blockIdx.x == 64 &&                                                            \
        (threadIdx.x == kWarps * 32 || threadIdx.x == (kWarps + 1) * 32 ||              \
         threadIdx.x == 32) && (slot) < 4096)                                          \
      g_trace[kid][threadIdx.x == 32 ? 1 : 0][(slot)] = clock64();                     \
  } while (0)
#else
#define SG_TRACE(kid, slot) \
  do {                      \
  } while (0)
#endif

__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
// 32 consecutive 32-bit TMEM columns of this thread's lane, one wait
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 consecutive 32-bit TMEM columns of this thread's lane <- v
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}
// 16 consecutive 32-bit TMEM columns of this thread's lane <- v
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]^T ("TS": A is read from TMEM, lane = row)
__device__ __forceinline__ void mma_tf32_ts(uint32_t dtmem, uint32_t atmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 2^x, flush-to-zero approximation (one MUFU op; 2^-inf = +0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// round a finite non-negative float to TF32, nearest, ties away (cvt.rna)
__device__ __forceinline__ float tf32_pos(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
constexpr float kLog2e = 1.4426950408889634f;
__device__ __forceinline__ uint32_t keep_mask(uint32_t j0, uint32_t limit) {
  // bit c set iff j0 + c < limit
  if (j0 >= limit) return 0u;
  const uint32_t n = limit - j0;
  return n >= 32 ? 0xffffffffu : (1u << n) - 1u;
}

// S = A . B^T over K = dpad into TMEM columns dcol (N = n columns), A and B
// K-major core-matrix tiles in shared memory
__device__ __forceinline__ void mma_scores_ss(uint32_t dcol, uint32_t a0, uint32_t b0, uint32_t dp,
                                              uint32_t n) {
  const uint32_t kcore = (dp / 4) * 128;
  const uint32_t id = instr_desc(128, n, false, false);
  for (uint32_t ks = 0; ks < dp / 8; ++ks)
    mma_tf32(dcol, smem_desc(a0 + ks * 256, 128, kcore), smem_desc(b0 + ks * 256, 128, kcore), id,
             ks > 0);
}
// barrier setup shared by the tensor-core kernels
__device__ __forceinline__ void sg_setup(uint32_t* tbase_s, uint32_t tcols, uint64_t* bars,
                                         int nbars, const uint32_t* counts) {
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(tbase_s, tcols);
  if (threadIdx.x == kWarps * 32) {
    for (int i = 0; i < nbars; ++i) bar_init(bars + i, counts[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

// SG2 (stats + mix, one pass): per tile, S = IR1 N^T block by block (128
// negatives per block: a tf32 MMA costs the same ~96 cycles at N = 64 or 128)
// with an online softmax per row -- the unnormalised weights W = 2^((S - mu)
// log2e) go to TMEM as the A operand of acc += W N; mu moves (and acc is
// rescaled) only when a block's max exceeds it by more than 2^8 in weight.
// At the end: c = mu log2e + log2 Z (SG3's weight offset), the loss
// (train.cpp:274) and mix = acc / Z - dst.  TMEM (512 columns): acc [0, 128),
// S buffers [128, 384), W [384, 512).  smem: IR1 tile (A of the S MMA), N
// blocks x2 (x1 when dpad = 128 would not fit), one N^T block (two 64-column
// core-matrix sub-tiles).
__global__ void __launch_bounds__(kThreadsSG, 1) sg2_mix_kernel(BatchArgs a, uint32_t tcols,
                                                                uint32_t nbuf) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t dp = a.dpad, k = a.k, kp = a.kpad, d = a.dim;
  const uint32_t tile_bytes = 128 * dp * 4, blk_bytes = kMixBlk * dp * 4;
  const uint32_t sub_bytes = 64 * dp * 4;    // one 64-negative N^T sub-tile
  unsigned char* sA = smem;
  unsigned char* sN = sA + tile_bytes;       // nbuf x N block
  unsigned char* sT = sN + nbuf * blk_bytes; // 1 x N^T block
  // 0 ld_a, 1-2 ld_n, 3 ld_t, 4-5 mma_s, 6-7 epi, 8 wrdy, 9 mma_w
  __shared__ uint64_t bars[10];
  __shared__ uint32_t tbase_s;
  // the two column halves' sums of each row, then 1 / Z (the dynamic buffers
  // leave ~3 KB of the 227)
  __shared__ float red_z[2][128];
  uint64_t *ld_a = bars, *ld_n = bars + 1, *ld_t = bars + 3, *mma_s = bars + 4, *epi = bars + 6,
           *wrdy = bars + 8, *mma_w = bars + 9;
  const uint32_t counts[10] = {1, 1, 1, 1, 1, 1, kWarps, kWarps, kWarps, 1};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const TileGeom g = tile_geom(a, blockIdx.x);
  sg_setup(&tbase_s, tcols, bars, 10, counts);
  SG_TRACE(1, 4090);
  const uint32_t tbase = tbase_s;
  const uint32_t nblk = kp / kMixBlk;
  const int q = warp & 3, hf = warp >> 2;
  const uint32_t row = q * 32 + lane;
  const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16);
  const uint64_t tile_p0 = g.c * a.chunk + (g.row0 - g.c * (uint64_t)a.tpc * 128);
  float mu = -INFINITY, zh = 0.f;  // epilogue: the row's online-softmax state
  // the tile's dst rows (mix = sum_j w_j n_j - dst, train.cpp:306-323): one
  // contiguous bulk copy of the prep kernel's tile-major copy into the N
  // blocks, once they are free (after the last S MMA; with one N buffer the
  // rows reach into the N^T block, so after the last mix MMA); ld_a's second
  // phase.  (A gather of the 128 rows here cost half of SG2's time.)
  const uint32_t dst_bytes = (g.valid * d * 4 + 15) & ~15u;
  unsigned char* sD = sN + 512;  // past the tail tile's overhang into sN
  auto load_dst = [&]() {
    if (!dst_bytes) return;
    bar_expect(ld_a, dst_bytes);
    bulk_load(sD, a.sh_D + g.row0 * d, dst_bytes, ld_a);
  };
  const unsigned char* gT =
      reinterpret_cast<const unsigned char*>(a.sh_BT) + g.c * (uint64_t)kp * dp * 4;
  auto load_t = [&](uint32_t b) {
    bar_expect(ld_t, blk_bytes);
    bulk_load(sT, gT + (uint64_t)b * blk_bytes, blk_bytes, ld_t);
  };
  if (warp == kWarps) {  // S issuer: the IR1 tile, the N blocks, S = IR1 N^T
    if (lane == 0) {
      const unsigned char* gA = reinterpret_cast<const unsigned char*>(a.sh_A) + g.row0 * dp * 4;
      const unsigned char* gN =
          reinterpret_cast<const unsigned char*>(a.sh_B) + g.c * (uint64_t)kp * dp * 4;
      auto load_n = [&](uint32_t b) {  // N block b into buffer b % nbuf
        const uint32_t i = b % nbuf;
        bar_expect(ld_n + i, blk_bytes);
        bulk_load(sN + i * blk_bytes, gN + (uint64_t)b * blk_bytes, blk_bytes, ld_n + i);
      };
      auto issue_s = [&](uint32_t b) {
        bar_wait(ld_n + b % nbuf, (b / nbuf) & 1);
        if (b >= 2) bar_wait(epi + (b & 1), ((b - 2) >> 1) & 1);
        tc_fence_after();
        mma_scores_ss(tbase + 128 + (b & 1) * kMixBlk, saddr(sA),
                      saddr(sN + (b % nbuf) * blk_bytes), dp, kMixBlk);
        mma_commit(mma_s + (b & 1));
      };
      bar_expect(ld_a, tile_bytes);
      bulk_load(sA, gA, tile_bytes, ld_a);
      for (uint32_t b = 0; b < nbuf && b < nblk; ++b) load_n(b);
      bar_wait(ld_a, 0);
      issue_s(0);
      for (uint32_t b = 0; b < nblk; ++b) {
        SG_TRACE(1, b * 8 + 0);
        if (nbuf == 2 && b + 1 < nblk) issue_s(b + 1);
        SG_TRACE(1, b * 8 + 1);
        bar_wait(mma_s + (b & 1), (b >> 1) & 1);
        if (b + nbuf < nblk) load_n(b + nbuf);  // S(b) is done with its buffer
        if (nbuf == 1 && b + 1 < nblk) issue_s(b + 1);
      }
      if (nbuf == 2) load_dst();
    }
  } else if (warp == kWarps + 1) {  // mix issuer: the N^T blocks, acc += W N
    // (a second issuing thread: its MMA chain interleaves with the S chain
    // on the tensor pipe instead of queueing behind it)
    if (lane == 0) {
      load_t(0);
      const uint32_t id = instr_desc(128, dp, false, false);
      for (uint32_t b = 0; b < nblk; ++b) {
        bar_wait(wrdy, b & 1);  // the epilogue wrote W(b)
        SG_TRACE(1, b * 8 + 2);
        bar_wait(ld_t, b & 1);
        tc_fence_after();
        // acc += W . N^T over the block's 128 negatives (two N^T sub-tiles)
        for (uint32_t ks = 0; ks < kMixBlk / 8; ++ks)
          mma_tf32_ts(tbase, tbase + 384 + ks * 8,
                      smem_desc(saddr(sT) + (ks >> 3) * sub_bytes + (ks & 7) * 256, 128, 16 * 128),
                      id, (b | ks) != 0);
        mma_commit(mma_w);
        SG_TRACE(1, b * 8 + 3);
        bar_wait(mma_w, b & 1);
        SG_TRACE(1, b * 8 + 4);
        if (b + 1 < nblk) load_t(b + 1);
      }
      if (nbuf != 2) load_dst();
    }
  } else {  // epilogue: warp half hf covers 64 of a block's 128 columns
    const bool valid = row < g.valid;
    // online softmax (train.cpp:262-274 restated): mu = the row's reference
    // max, zh = this half's sum of 2^((s - mu) log2e); W = the unnormalised
    // weights, the accumulator rescaled when mu moves and divided by Z at the end
    for (uint32_t nb = 0; nb < nblk; ++nb) {
      SG_TRACE(1, nb * 8 + 0);
      bar_wait(mma_s + (nb & 1), (nb >> 1) & 1);
      tc_fence_after();
      SG_TRACE(1, nb * 8 + 1);
      const uint32_t scol0 = 128 + (nb & 1) * kMixBlk + hf * 64;
      const uint32_t scol1 = 128 + (nb & 1) * kMixBlk + (hf ^ 1) * 64;
      const uint32_t j0 = nb * kMixBlk + hf * 64, j1 = nb * kMixBlk + (hf ^ 1) * 64;
      // the block's row max over all 128 columns: the other half's 64 are read
      // too (warps q and q + 4 share the rows), so both warps of the pair
      // agree on it with no exchange
      float bm = -INFINITY;
      for (int part = 0; part < 2; ++part) {
        float x[32];
        tmem_ld32(lane_addr + scol1 + 32 * part, x);
        const uint32_t kx = valid ? keep_mask(j1 + 32 * part, k) : 0u;
#pragma unroll
        for (int c = 0; c < 32; ++c) bm = fmaxf(bm, (kx >> c) & 1u ? x[c] : -INFINITY);
      }
      float v[64];
      tmem_ld32(lane_addr + scol0, v);
      tmem_ld32(lane_addr + scol0 + 32, v + 32);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(epi + (nb & 1));  // the S buffer is free
      const uint32_t keep0 = valid ? keep_mask(j0, k) : 0u;
      const uint32_t keep1 = valid ? keep_mask(j0 + 32, k) : 0u;
      const bool full = (keep0 & keep1) == 0xffffffffu;
      if (full) {
#pragma unroll
        for (int c = 0; c < 64; ++c) bm = fmaxf(bm, v[c]);
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          bm = fmaxf(bm, ((c < 32 ? keep0 : keep1) >> (c & 31)) & 1u ? v[c] : -INFINITY);
      }
      const float bmax = bm;
      // the reference max moves only when the block's max exceeds it by more
      // than 2^8 in weight, so the accumulator is rarely rescaled; both warps
      // of the row pair decide alike
      const float mu_new =
          (mu == -INFINITY || (bmax - mu) * kLog2e > 8.f) ? bmax : mu;
      const float f = mu == -INFINITY ? 0.f : ex2((mu - mu_new) * kLog2e);
      const bool rescale = __any_sync(0xffffffffu, mu != -INFINITY && mu_new != mu);
      mu = mu_new;
      const float ml2 = mu == -INFINITY ? 0.f : mu * kLog2e;
      float z0 = 0.f, z1 = 0.f;
      if (full) {
#pragma unroll
        for (int c = 0; c < 64; c += 2) {
          const float e0 = ex2(__fmaf_rn(v[c], kLog2e, -ml2));
          const float e1 = ex2(__fmaf_rn(v[c + 1], kLog2e, -ml2));
          z0 += e0;
          z1 += e1;
          v[c] = tf32_pos(e0);
          v[c + 1] = tf32_pos(e1);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const bool kc = ((c < 32 ? keep0 : keep1) >> (c & 31)) & 1u;
          const float e = kc ? ex2(__fmaf_rn(v[c], kLog2e, -ml2)) : 0.f;
          z0 += e;
          v[c] = tf32_pos(e);
        }
      }
      zh = zh * f + (z0 + z1);
      SG_TRACE(1, nb * 8 + 2);
      if (nb >= 1) bar_wait(mma_w, (nb - 1) & 1);  // W and the accumulator free again
      tc_fence_after();
      SG_TRACE(1, nb * 8 + 3);
      if (rescale) {  // this half's accumulator columns, scaled to the new reference
        const uint32_t c0 = hf * 64, c1 = hf ? dp : (dp < 64 ? dp : 64);
        for (uint32_t cc = c0; cc < c1; cc += 16) {
          float x[16];
          tmem_ld16(lane_addr + cc, x);
#pragma unroll
          for (int e = 0; e < 16; ++e) x[e] *= f;
          tmem_st16(lane_addr + cc, x);
        }
      }
      tmem_st32(lane_addr + 384 + hf * 64, v);
      tmem_st32(lane_addr + 384 + hf * 64 + 32, v + 32);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(wrdy);
      SG_TRACE(1, nb * 8 + 4);
    }
    red_z[hf][row] = zh;
  }
  SG_TRACE(1, 4001);
  __syncthreads();
  SG_TRACE(1, 4002);
  if (warp < 4 && row < g.valid) {  // the row's statistics: the weights' offset and the loss
    const float Z = red_z[0][row] + red_z[1][row];
    const uint64_t tr = g.row0 + row;
    const uint64_t p = tile_p0 + row;
    a.sh_rowc[tr] = (float)((double)mu * (double)kLog2e + log2((double)Z));
    a.loss[p] = -(a.sh_pos[p] - ((double)mu + log((double)Z)));  // train.cpp:274
    red_z[0][row] = 1.f / Z;
  }
  bar_wait(mma_w, (nblk - 1) & 1);
  SG_TRACE(1, 4003);
  tc_fence_after();
  // mix accumulator -> shared tile (the IR1 tile, overhanging into the free N
  // blocks by dpad floats); odd row stride: lanes (rows) hit distinct banks
  float* out = reinterpret_cast<float*>(sA);
  const uint32_t ts = dp + 1;
  if (warp < kWarps) {
    const uint32_t c0 = hf * 64, c1 = hf ? dp : (dp < 64 ? dp : 64);
    for (uint32_t cc = c0; cc < c1; cc += 16) {
      float v[16];
      tmem_ld16(lane_addr + cc, v);
#pragma unroll
      for (int e = 0; e < 16; ++e) out[row * ts + cc + e] = v[e];
    }
  }
  SG_TRACE(1, 4004);
  tc_fence_before();
  __syncthreads();
  SG_TRACE(1, 4005);
  // mix rows in FP64, coalesced, by all ten warps (the tail is latency-bound:
  // two rows per step keep eight independent chains per lane; staging them
  // for bulk stores measured slower)
  if (dst_bytes) {
    bar_wait(ld_a, 1);
    SG_TRACE(1, 4006);
    const float* dsts = reinterpret_cast<const float*>(sD);
    constexpr uint32_t kAll = kWarps + 2;
    for (uint32_t r = warp; r < g.valid; r += 2 * kAll) {
      const uint32_t r2 = r + kAll;
      const bool two = r2 < g.valid;
      const float inv = red_z[0][r], inv2 = two ? red_z[0][r2] : 0.f;
      double* mx = a.mix + (tile_p0 + r) * d;
      double* mx2 = a.mix + (tile_p0 + r2) * d;
      for (uint32_t e = lane; e < d; e += 32) {
        const float o = out[r * ts + e], t = dsts[r * d + e];
        const float o2 = two ? out[r2 * ts + e] : 0.f, t2 = two ? dsts[r2 * d + e] : 0.f;
        mx[e] = (double)(o * inv) - (double)t;
        if (two) mx2[e] = (double)(o2 * inv2) - (double)t2;
      }
    }
    SG_TRACE(1, 4007);
  }
  __syncthreads();
  SG_TRACE(1, 4091);
  if (warp == 0) tmem_free(tbase, tcols);
}

// SG3: per (chunk, 128 negatives): G = W^T IR1 over the chunk's positives in
// 128-positive slices; S^T = N IR1^T is recomputed per slice (M = the 128
// negatives, N = 128 positives).  TMEM (512 columns): G [0, 128), S^T buffers
// [128, 384), W^T [384, 512) (A of the G MMA).  smem: the negative block (A of
// the S^T MMA), IR1 tiles x2 (x1 when dpad = 128 would not fit), one IR1^T
// slice pair (two 64-column core-matrix sub-tiles).
__global__ void __launch_bounds__(kThreadsSG, 1) sg3_grad_kernel(BatchArgs a, uint32_t tcols,
                                                                 uint32_t nbuf) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t dp = a.dpad, k = a.k, kp = a.kpad, d = a.dim;
  const uint32_t nblk_bytes = 128 * dp * 4, sl_bytes = kGradSlice * dp * 4;
  const uint32_t sub_bytes = 64 * dp * 4;  // one 64-positive IR1^T sub-tile
  unsigned char* sN = smem;
  unsigned char* sA = sN + nblk_bytes;      // nbuf x IR1 tile
  unsigned char* sT = sA + nbuf * sl_bytes; // 1 x IR1^T slice
  // 0 ld_n, 1-2 ld_a, 3 ld_t, 4-5 mma_s, 6-7 epi, 8 wrdy, 9 mma_w
  __shared__ uint64_t bars[10];
  __shared__ uint32_t tbase_s;
  uint64_t *ld_n = bars, *ld_a = bars + 1, *ld_t = bars + 3, *mma_s = bars + 4, *epi = bars + 6,
           *wrdy = bars + 8, *mma_w = bars + 9;
  const uint32_t counts[10] = {1, 1, 1, 1, 1, 1, kWarps, kWarps, kWarps, 1};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, hf = warp >> 2;
  const uint32_t row = q * 32 + lane;  // negative n0 + row
  const uint32_t nbpc = kp / 128;
  const uint64_t c = blockIdx.x / nbpc;
  const uint32_t n0 = (blockIdx.x - c * nbpc) * 128;
  const uint64_t left = a.P - c * a.chunk;
  const uint64_t chunk_rows = left < a.chunk ? left : a.chunk;
  const uint32_t nsl = (uint32_t)((chunk_rows + kGradSlice - 1) / kGradSlice);
  const uint64_t crow0 = c * (uint64_t)a.tpc * 128;
  sg_setup(&tbase_s, tcols, bars, 10, counts);
  SG_TRACE(2, 4090);
  const uint32_t tbase = tbase_s;
  const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16);
  const unsigned char* gT = reinterpret_cast<const unsigned char*>(a.sh_AT) + crow0 * dp * 4;
  auto load_t = [&](uint32_t s) {
    bar_expect(ld_t, sl_bytes);
    bulk_load(sT, gT + (uint64_t)s * sl_bytes, sl_bytes, ld_t);
  };
  if (warp == kWarps) {  // S issuer: the negative block, the IR1 slices, S^T = N IR1^T
    if (lane == 0) {
      const unsigned char* gA = reinterpret_cast<const unsigned char*>(a.sh_A) + crow0 * dp * 4;
      const unsigned char* gN =
          reinterpret_cast<const unsigned char*>(a.sh_B) + (c * (uint64_t)kp + n0) * dp * 4;
      auto load_a = [&](uint32_t s) {
        const uint32_t i = s % nbuf;
        bar_expect(ld_a + i, sl_bytes);
        bulk_load(sA + i * sl_bytes, gA + (uint64_t)s * sl_bytes, sl_bytes, ld_a + i);
      };
      auto issue_s = [&](uint32_t s) {
        bar_wait(ld_a + s % nbuf, (s / nbuf) & 1);
        if (s >= 2) bar_wait(epi + (s & 1), ((s - 2) >> 1) & 1);
        tc_fence_after();
        mma_scores_ss(tbase + 128 + (s & 1) * kGradSlice, saddr(sN),
                      saddr(sA + (s % nbuf) * sl_bytes), dp, kGradSlice);
        mma_commit(mma_s + (s & 1));
      };
      bar_expect(ld_n, nblk_bytes);
      bulk_load(sN, gN, nblk_bytes, ld_n);
      for (uint32_t s = 0; s < nbuf && s < nsl; ++s) load_a(s);
      bar_wait(ld_n, 0);
      issue_s(0);
      SG_TRACE(2, 4000);
      for (uint32_t s = 0; s < nsl; ++s) {
        SG_TRACE(2, s * 8 + 0);
        if (nbuf == 2 && s + 1 < nsl) issue_s(s + 1);
        SG_TRACE(2, s * 8 + 1);
        bar_wait(mma_s + (s & 1), (s >> 1) & 1);
        SG_TRACE(2, s * 8 + 2);
        if (s + nbuf < nsl) load_a(s + nbuf);
        if (nbuf == 1 && s + 1 < nsl) issue_s(s + 1);
      }
    }
  } else if (warp == kWarps + 1) {  // G issuer: the IR1^T slices, G += W^T IR1
    if (lane == 0) {
      load_t(0);
      const uint32_t id = instr_desc(128, dp, false, false);
      for (uint32_t s = 0; s < nsl; ++s) {
        bar_wait(wrdy, s & 1);
        SG_TRACE(2, s * 8 + 3);
        bar_wait(ld_t, s & 1);
        SG_TRACE(2, s * 8 + 4);
        tc_fence_after();
        // G += W^T . IR1 over the slice's 128 positives (two IR1^T sub-tiles)
        for (uint32_t ks = 0; ks < kGradSlice / 8; ++ks)
          mma_tf32_ts(tbase, tbase + 384 + ks * 8,
                      smem_desc(saddr(sT) + (ks >> 3) * sub_bytes + (ks & 7) * 256, 128, 16 * 128),
                      id, (s | ks) != 0);
        mma_commit(mma_w);
        bar_wait(mma_w, s & 1);
        SG_TRACE(2, s * 8 + 5);
        if (s + 1 < nsl) load_t(s + 1);
      }
    }
  } else {  // epilogue: row = negative, warp half hf covers 64 of the slice's positives
    const bool nvalid = n0 + row < k;
    // the offsets c of this half's 64 positives of slice s: lane i holds
    // positives i and 32 + i; loaded one slice ahead (their latency overlaps
    // the wait for the slice's MMA)
    auto load_c = [&](uint32_t s, float& c0, float& c1) {
      const uint64_t pq0 = (uint64_t)s * kGradSlice + hf * 64 + lane, pq1 = pq0 + 32;
      c0 = pq0 < chunk_rows ? a.sh_rowc[crow0 + pq0] : 0.f;
      c1 = pq1 < chunk_rows ? a.sh_rowc[crow0 + pq1] : 0.f;
    };
    float cn0, cn1;
    load_c(0, cn0, cn1);
    for (uint32_t s = 0; s < nsl; ++s) {
      const uint64_t pq0 = (uint64_t)s * kGradSlice + hf * 64 + lane, pq1 = pq0 + 32;
      const bool pv0 = pq0 < chunk_rows, pv1 = pq1 < chunk_rows;
      const float c0 = cn0, c1 = cn1;
      if (s + 1 < nsl) load_c(s + 1, cn0, cn1);
      const uint32_t pm0 = __ballot_sync(0xffffffffu, pv0);  // every lane: no divergent vote
      const uint32_t pm1 = __ballot_sync(0xffffffffu, pv1);
      const uint32_t keep0 = nvalid ? pm0 : 0u, keep1 = nvalid ? pm1 : 0u;
      SG_TRACE(2, s * 8 + 0);
      bar_wait(mma_s + (s & 1), (s >> 1) & 1);
      SG_TRACE(2, s * 8 + 1);
      tc_fence_after();
      const uint32_t scol0 = 128 + (s & 1) * kGradSlice + hf * 64;
      float v[32], w0[32], w1[32];
      tmem_ld32(lane_addr + scol0, v);
#pragma unroll
      for (int cc = 0; cc < 32; ++cc) {
        const float e = ex2(__fmaf_rn(v[cc], kLog2e, -__shfl_sync(0xffffffffu, c0, cc)));
        w0[cc] = (keep0 >> cc) & 1u ? tf32_pos(e) : 0.f;
      }
      tmem_ld32(lane_addr + scol0 + 32, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(epi + (s & 1));
#pragma unroll
      for (int cc = 0; cc < 32; ++cc) {
        const float e = ex2(__fmaf_rn(v[cc], kLog2e, -__shfl_sync(0xffffffffu, c1, cc)));
        w1[cc] = (keep1 >> cc) & 1u ? tf32_pos(e) : 0.f;
      }
      SG_TRACE(2, s * 8 + 2);
      if (s >= 1) bar_wait(mma_w, (s - 1) & 1);  // W^T free again
      SG_TRACE(2, s * 8 + 3);
      tc_fence_after();
      tmem_st32(lane_addr + 384 + hf * 64, w0);
      tmem_st32(lane_addr + 384 + hf * 64 + 32, w1);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(wrdy);
      SG_TRACE(2, s * 8 + 4);
    }
  }
  __syncthreads();
  bar_wait(mma_w, (nsl - 1) & 1);
  tc_fence_after();
  // G rows: TMEM -> the free negative block as compact rows (the chunk block's
  // rows are contiguous in sh_G), then one bulk store (a row-by-row copy
  // loop here was latency-bound: ~9k cycles of 8 warps)
  float* out = reinterpret_cast<float*>(sN);
  const uint32_t nrows = k > n0 ? (k - n0 < 128 ? k - n0 : 128) : 0;
  const uint32_t g_bytes = nrows * d * 4;
  float* gdst = a.sh_G + (c * (uint64_t)kp + n0) * d;
  const bool bulk = g_bytes && (g_bytes & 15) == 0 && ((c * (uint64_t)kp + n0) * d * 4 & 15) == 0;
  if (warp < kWarps) {  // (tcgen05.ld is warp-collective: every lane loads, rows < nrows store)
    const uint32_t c0 = hf * 64, c1 = hf ? dp : (dp < 64 ? dp : 64);
    float* o = bulk ? out + row * d : gdst + (uint64_t)row * d;
    for (uint32_t cc = c0; cc < c1; cc += 16) {
      float v[16];
      tmem_ld16(lane_addr + cc, v);
      if (row < nrows) {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (cc + e < d) o[cc + e] = v[e];
      }
    }
    if (bulk) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if (bulk && threadIdx.x == 0) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
                 "r"(saddr(out)), "r"(g_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // shared memory reusable
  }
  __syncthreads();
  SG_TRACE(2, 4091);
  if (warp == 0) tmem_free(tbase, tcols);
}


// SG3, persistent (two IR1 slice buffers fit): one CTA per SM walks the (chunk,
// 128-negative block) items blockIdx.x, + gridDim.x, ... as one stream of
// slices, so a slice's loads, MMAs and epilogue overlap across item
// boundaries: the next item's IR1 slices and IR1^T slice are prefetched by
// the ring as usual, its negative block loads as soon as the last S^T MMA of
// the current item is done, and the epilogue drains G straight from TMEM to
// global memory while the next item's first S^T MMA runs (acc_free orders
// the next item's first G MMA after the drain).
struct Sg3Item {
  uint64_t c, chunk_rows, crow0;
  uint32_t n0, nsl;
};
__device__ __forceinline__ Sg3Item sg3_item(const BatchArgs& a, uint64_t w) {
  const uint32_t nbpc = a.kpad / 128;
  Sg3Item it;
  it.c = w / nbpc;
  it.n0 = (uint32_t)(w - it.c * nbpc) * 128;
  const uint64_t left = a.P - it.c * a.chunk;
  it.chunk_rows = left < a.chunk ? left : a.chunk;
  it.nsl = (uint32_t)((it.chunk_rows + kGradSlice - 1) / kGradSlice);
  it.crow0 = it.c * (uint64_t)a.tpc * 128;
  return it;
}
struct Sg3Cursor {  // (item, slice) of a CTA's slice stream
  uint64_t w, nitems;
  uint32_t s, ii, step;
  Sg3Item it;
  bool valid;
  __device__ void start(const BatchArgs& a, uint64_t w0, uint32_t stride, uint64_t n) {
    w = w0;
    nitems = n;
    s = 0;
    ii = 0;
    step = stride;
    valid = w < nitems;
    if (valid) it = sg3_item(a, w);
  }
  __device__ void advance(const BatchArgs& a) {
    if (!valid) return;
    if (++s < it.nsl) return;
    s = 0;
    ++ii;
    w += step;
    valid = w < nitems;
    if (valid) it = sg3_item(a, w);
  }
};

__global__ void __launch_bounds__(kThreadsSG, 1) sg3_persistent_kernel(BatchArgs a, uint32_t tcols,
                                                                       uint64_t nitems) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t dp = a.dpad, k = a.k, kp = a.kpad, d = a.dim;
  const uint32_t nblk_bytes = 128 * dp * 4, sl_bytes = kGradSlice * dp * 4;
  const uint32_t sub_bytes = 64 * dp * 4;  // one 64-positive IR1^T sub-tile
  unsigned char* sN = smem;
  unsigned char* sA = sN + nblk_bytes;   // 2 x IR1 slice
  unsigned char* sT = sA + 2 * sl_bytes;  // 1 x IR1^T slice
  // 0 ld_n, 1-2 ld_a, 3 ld_t, 4-5 mma_s, 6-7 epi, 8 wrdy, 9 mma_w, 10 acc_free
  __shared__ uint64_t bars[11];
  __shared__ uint32_t tbase_s;
  uint64_t *ld_n = bars, *ld_a = bars + 1, *ld_t = bars + 3, *mma_s = bars + 4, *epi = bars + 6,
           *wrdy = bars + 8, *mma_w = bars + 9, *acc_free = bars + 10;
  const uint32_t counts[11] = {1, 1, 1, 1, 1, 1, kWarps, kWarps, kWarps, 1, kWarps};
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, hf = warp >> 2;
  const uint32_t row = q * 32 + lane;  // negative n0 + row
  sg_setup(&tbase_s, tcols, bars, 11, counts);
  SG_TRACE(2, 4090);
  const uint32_t tbase = tbase_s;
  const uint32_t lane_addr = tbase + ((uint32_t)(q * 32) << 16);
  const unsigned char* gA0 = reinterpret_cast<const unsigned char*>(a.sh_A);
  const unsigned char* gT0 = reinterpret_cast<const unsigned char*>(a.sh_AT);
  const unsigned char* gN0 = reinterpret_cast<const unsigned char*>(a.sh_B);
  Sg3Cursor first;
  first.start(a, blockIdx.x, gridDim.x, nitems);
  if (warp == kWarps) {  // S issuer: negative blocks, IR1 slices, S^T = N IR1^T
    if (lane == 0) {
      auto load_n = [&](const Sg3Cursor& cu) {
        bar_expect(ld_n, nblk_bytes);
        bulk_load(sN, gN0 + (cu.it.c * (uint64_t)kp + cu.it.n0) * dp * 4, nblk_bytes, ld_n);
      };
      auto load_a = [&](const Sg3Cursor& cu, uint32_t g) {
        bar_expect(ld_a + (g & 1), sl_bytes);
        bulk_load(sA + (g & 1) * sl_bytes, gA0 + (cu.it.crow0 * dp * 4 + (uint64_t)cu.s * sl_bytes),
                  sl_bytes, ld_a + (g & 1));
      };
      auto issue_s = [&](const Sg3Cursor& cu, uint32_t g) {
        bar_wait(ld_a + (g & 1), (g >> 1) & 1);
        if (g >= 2) bar_wait(epi + (g & 1), ((g - 2) >> 1) & 1);
        if (cu.s == 0) bar_wait(ld_n, cu.ii & 1);
        tc_fence_after();
        mma_scores_ss(tbase + 128 + (g & 1) * kGradSlice, saddr(sN), saddr(sA + (g & 1) * sl_bytes),
                      dp, kGradSlice);
        mma_commit(mma_s + (g & 1));
      };
      Sg3Cursor cur = first, ld = first;
      load_n(cur);
      load_a(ld, 0);
      ld.advance(a);
      if (ld.valid) {
        load_a(ld, 1);
        ld.advance(a);
      }
      issue_s(cur, 0);
      Sg3Cursor nx = cur;
      nx.advance(a);
      for (uint32_t g = 0; cur.valid; ++g) {
        SG_TRACE(2, (g & 511) * 8 + 0);
        const bool crossing = nx.valid && nx.ii != cur.ii;
        if (nx.valid && !crossing) issue_s(nx, g + 1);
        bar_wait(mma_s + (g & 1), (g >> 1) & 1);  // S^T(g) done: its IR1 slot (and sN) free
        SG_TRACE(2, (g & 511) * 8 + 1);
        if (crossing) {  // the next item's negative block, then its first S^T MMA
          load_n(nx);
          issue_s(nx, g + 1);
        }
        if (ld.valid) {
          load_a(ld, g + 2);
          ld.advance(a);
        }
        cur = nx;
        nx.advance(a);
      }
    }
  } else if (warp == kWarps + 1) {  // G issuer: IR1^T slices, G += W^T IR1
    if (lane == 0) {
      auto load_t = [&](const Sg3Cursor& cu) {
        bar_expect(ld_t, sl_bytes);
        bulk_load(sT, gT0 + (cu.it.crow0 * dp * 4 + (uint64_t)cu.s * sl_bytes), sl_bytes, ld_t);
      };
      const uint32_t id = instr_desc(128, dp, false, false);
      Sg3Cursor cur = first;
      load_t(cur);
      for (uint32_t g = 0; cur.valid; ++g) {
        bar_wait(wrdy, g & 1);
        bar_wait(ld_t, g & 1);
        if (cur.s == 0 && cur.ii > 0) bar_wait(acc_free, (cur.ii - 1) & 1);  // G drained
        SG_TRACE(2, (g & 511) * 8 + 3);
        tc_fence_after();
        for (uint32_t ks = 0; ks < kGradSlice / 8; ++ks)
          mma_tf32_ts(tbase, tbase + 384 + ks * 8,
                      smem_desc(saddr(sT) + (ks >> 3) * sub_bytes + (ks & 7) * 256, 128, 16 * 128),
                      id, (cur.s | ks) != 0);
        mma_commit(mma_w);
        bar_wait(mma_w, g & 1);
        SG_TRACE(2, (g & 511) * 8 + 5);
        cur.advance(a);
        if (cur.valid) load_t(cur);
      }
    }
  } else {  // epilogue: row = negative, warp half hf covers 64 of the slice's positives
    auto load_c = [&](const Sg3Cursor& cu, float& c0, float& c1) {
      const uint64_t pq0 = (uint64_t)cu.s * kGradSlice + hf * 64 + lane, pq1 = pq0 + 32;
      c0 = pq0 < cu.it.chunk_rows ? a.sh_rowc[cu.it.crow0 + pq0] : 0.f;
      c1 = pq1 < cu.it.chunk_rows ? a.sh_rowc[cu.it.crow0 + pq1] : 0.f;
    };
    Sg3Cursor cur = first;
    float cn0 = 0.f, cn1 = 0.f;
    if (cur.valid) load_c(cur, cn0, cn1);
    for (uint32_t g = 0; cur.valid; ++g) {
      const Sg3Item it = cur.it;
      const bool nvalid = it.n0 + row < k;
      const uint64_t pq0 = (uint64_t)cur.s * kGradSlice + hf * 64 + lane, pq1 = pq0 + 32;
      const bool pv0 = pq0 < it.chunk_rows, pv1 = pq1 < it.chunk_rows;
      const float c0 = cn0, c1 = cn1;
      Sg3Cursor nx = cur;
      nx.advance(a);
      if (nx.valid) load_c(nx, cn0, cn1);
      const uint32_t pm0 = __ballot_sync(0xffffffffu, pv0);
      const uint32_t pm1 = __ballot_sync(0xffffffffu, pv1);
      const uint32_t keep0 = nvalid ? pm0 : 0u, keep1 = nvalid ? pm1 : 0u;
      bar_wait(mma_s + (g & 1), (g >> 1) & 1);
      tc_fence_after();
      const uint32_t scol0 = 128 + (g & 1) * kGradSlice + hf * 64;
      float v[32], w0[32], w1[32];
      tmem_ld32(lane_addr + scol0, v);
#pragma unroll
      for (int cc = 0; cc < 32; ++cc) {
        const float e = ex2(__fmaf_rn(v[cc], kLog2e, -__shfl_sync(0xffffffffu, c0, cc)));
        w0[cc] = (keep0 >> cc) & 1u ? tf32_pos(e) : 0.f;
      }
      tmem_ld32(lane_addr + scol0 + 32, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(epi + (g & 1));
#pragma unroll
      for (int cc = 0; cc < 32; ++cc) {
        const float e = ex2(__fmaf_rn(v[cc], kLog2e, -__shfl_sync(0xffffffffu, c1, cc)));
        w1[cc] = (keep1 >> cc) & 1u ? tf32_pos(e) : 0.f;
      }
      if (g >= 1) bar_wait(mma_w, (g - 1) & 1);  // W^T free again
      tc_fence_after();
      tmem_st32(lane_addr + 384 + hf * 64, w0);
      tmem_st32(lane_addr + 384 + hf * 64 + 32, w1);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(wrdy);
      SG_TRACE(2, (g & 511) * 8 + 4);
      if (cur.s + 1 == it.nsl) {  // the item's last slice: G -> global rows, then acc_free
        bar_wait(mma_w, g & 1);
        tc_fence_after();
        const uint32_t nrows = k > it.n0 ? (k - it.n0 < 128 ? k - it.n0 : 128) : 0;
        float* grow = a.sh_G + (it.c * (uint64_t)kp + it.n0 + row) * d;
        const uint32_t c0r = hf * 64, c1r = hf ? dp : (dp < 64 ? dp : 64);
        for (uint32_t cc = c0r; cc < c1r; cc += 16) {
          float x[16];
          tmem_ld16(lane_addr + cc, x);  // warp-collective: every lane loads
          if (row < nrows) {
            if ((d & 3) == 0 && cc + 16 <= d) {
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(grow + cc + e) =
                    make_float4(x[e], x[e + 1], x[e + 2], x[e + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (cc + e < d) grow[cc + e] = x[e];
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(acc_free);
      }
      cur = nx;
    }
  }
  __syncthreads();
  SG_TRACE(2, 4091);
  if (warp == 0) tmem_free(tbase, tcols);
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  LGD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

#ifdef LGD_TRACE
extern "C" int lgd_debug_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)) == cudaSuccess ? 0 : 4;
}
#endif

// LGD_SG3_CLASSIC=1: one CTA per item (A/B against the persistent SG3)
static const bool g_sg3_classic = [] {
  const char* e = std::getenv("LGD_SG3_CLASSIC");
  return e && std::strtol(e, nullptr, 10) != 0;
}();

SharedShape shared_shape(uint32_t dim, uint32_t k, uint32_t chunk, uint64_t P) {
  SharedShape s{};
  s.dpad = (dim + 15) & ~15u;
  s.kpad = (k + 127) & ~127u;
  s.tpc = (chunk + 127) / 128;
  s.nch = chunk ? (P + chunk - 1) / chunk : 0;
  return s;
}

size_t shared_smem_bytes(uint32_t dpad) {
  const size_t t = 128ull * dpad * 4;
  const size_t sg2 = t + 2 * (size_t)kMixBlk * dpad * 4;
  const size_t sg3 = t + 2 * (size_t)kGradSlice * dpad * 4;
  return sg2 > sg3 ? sg2 : sg3;
}

void launch_shared_scores(const BatchArgs& a, cudaStream_t st) {
  const uint64_t rows = a.nch * (uint64_t)a.tpc * 128;
  const uint32_t dp = a.dpad;
  const size_t psm = (size_t)kPrepRows * (dp + 4) * 4;
  switch (a.kind) {
    case 0:
      shared_prep_kernel<0><<<(unsigned)(rows / kPrepRows), 256, psm, st>>>(a);
      break;
    case 1:
      shared_prep_kernel<1><<<(unsigned)(rows / kPrepRows), 256, psm, st>>>(a);
      break;
    default:
      shared_prep_kernel<2><<<(unsigned)(rows / kPrepRows), 256, psm, st>>>(a);
      break;
  }
  LGD_LAUNCH_CHECK();
  shared_gather_kernel<<<(unsigned)(a.nch * (uint64_t)a.kpad / kPrepRows), 256, psm, st>>>(a);
  LGD_LAUNCH_CHECK();
  const size_t t = 128ull * dp * 4;
  // SG2: two N buffers when they fit next to the tile and the N^T block
  const size_t mblk = (size_t)kMixBlk * dp * 4;
  const uint32_t nbuf2 = t + 3 * mblk <= 227 * 1024 ? 2 : 1;
  const size_t sm2 = t + (nbuf2 + 1) * mblk;
  const size_t gsl = (size_t)kGradSlice * dp * 4;
  const uint32_t nbuf3 = t + 3 * gsl <= 227 * 1024 ? 2 : 1;
  const size_t sm3 = t + (nbuf3 + 1) * gsl;
  static size_t set2[kMaxDevices], set3[kMaxDevices];  // grow only
  const int dev = current_device();
  if (sm2 > set2[dev]) set_smem(sg2_mix_kernel, set2[dev] = sm2);
  if (sm3 > set3[dev]) set_smem(sg3_grad_kernel, set3[dev] = sm3);
  const unsigned tiles = (unsigned)(a.nch * a.tpc);
  const uint32_t tcols = 512;   // + the TMEM A operands at 256 and 384
  sg2_mix_kernel<<<tiles, kThreadsSG, sm2, st>>>(a, tcols, nbuf2);
  LGD_LAUNCH_CHECK();
  const uint64_t items3 = a.nch * (a.kpad / 128);
  if (nbuf3 == 2 && !g_sg3_classic) {  // persistent: one CTA per SM over the item stream
    static size_t setp[kMaxDevices];
    if (sm3 > setp[dev]) set_smem(sg3_persistent_kernel, setp[dev] = sm3);
    const unsigned grid3 = (unsigned)(items3 < (uint64_t)a.sm_count ? items3 : a.sm_count);
    sg3_persistent_kernel<<<grid3, kThreadsSG, sm3, st>>>(a, tcols, items3);
  } else {
    sg3_grad_kernel<<<(unsigned)items3, kThreadsSG, sm3, st>>>(a, tcols, nbuf3);
  }
  LGD_LAUNCH_CHECK();
}

}  // namespace lgd
