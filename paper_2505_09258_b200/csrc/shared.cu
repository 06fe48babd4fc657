// shared.cu -- shared-negative chunks on the 5th-generation tensor cores.
//
// Mode: every run of C consecutive
// positives of a batch (a "chunk") shares the same k negatives, drawn from the
// bucket stream right where the reference draws its P k per-positive ones
// (ceil(P / C) k draws per batch).  The reference math on the expanded
// negative list is the oracle; scores are a dense chunk x negatives x dim
// contraction, computed here with tcgen05.mma kind::tf32 (FP32 accumulate in
// TMEM), in three kernels that never materialise the P x k weight matrix:
//
//   SG1 stats   per 128-positive tile: S = IR1 N^T block by block (64
//               negatives), online row max / sum of exp  ->  M_p, 1/Z_p, loss_p
//   SG2 mix     per tile: recompute S, W = exp(S - M) / Z into shared memory,
//               mix += W N on the tensor core
//   SG3 grad    per (chunk, 128 negatives): S^T = N IR1^T recomputed per
//               64-positive slice, W^T into shared memory, G += W^T IR1
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
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "train.cuh"

namespace lgd {

namespace {

constexpr int kThreads = 128;  // 4 warps: TMEM lanes 0..127 = tile rows
constexpr int kNegBlk = 64;    // negatives per S block (SG1 / SG2)
constexpr int kPosSlice = 64;  // positives per slice (SG3)

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
// generic-proxy shared-memory writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

__device__ __forceinline__ uint32_t cm_offset(uint32_t r, uint32_t c, uint32_t cols) {
  return ((r >> 3) * (cols >> 2) + (c >> 2)) * 128 + (r & 7) * 16 + (c & 3) * 4;
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
// One warp per padded tile row: IR1 (TF32) in the core-matrix layout, the
// positive score in FP64, snap = src row, mix = -dst, the dst / src
// contribution items and the relation key.  Padding rows are zero.
template <int KIND>
__global__ void __launch_bounds__(256) shared_prep_kernel(BatchArgs a) {
  const uint64_t row = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t C = a.chunk, d = a.dim, dp = a.dpad, h = d / 2;
  const uint64_t rows_per_chunk = (uint64_t)a.tpc * 128;
  if (row >= a.nch * rows_per_chunk) return;
  const uint64_t c = row / rows_per_chunk, r = row - c * rows_per_chunk;
  const uint64_t p = c * C + r;
  const bool valid = r < C && p < a.P;
  unsigned char* tile = reinterpret_cast<unsigned char*>(a.sh_A) + (row >> 7) * 128ull * dp * 4;
  unsigned char* tslice = reinterpret_cast<unsigned char*>(a.sh_AT) + (row >> 6) * 64ull * dp * 4;
  const uint32_t rr = (uint32_t)(row & 127), rt = (uint32_t)(row & 63);
  if (!valid) {
    for (uint32_t i = lane; i < dp; i += 32) {
      *reinterpret_cast<float*>(tile + cm_offset(rr, i, dp)) = 0.f;
      *reinterpret_cast<float*>(tslice + cm_offset(i, rt, 64)) = 0.f;
    }
    return;
  }
  const uint32_t s = a.edges[3 * p], rel = a.edges[3 * p + 1], t = a.edges[3 * p + 2];
  const float* srow = a.theta + (size_t)s * d;
  const float* rrow = KIND != 0 ? a.rel_theta + (size_t)rel * d : nullptr;
  const float* drow = a.theta + (size_t)t * d;
  double pos = 0.0;
  for (uint32_t i = lane; i < dp; i += 32) {
    double x = 0.0;
    if (i < d) {
      if (KIND == 2) {
        const uint32_t j = i < h ? i : i - h;
        const double sr = srow[j], si = srow[j + h], qr = rrow[j], qi = rrow[j + h];
        x = i < h ? sr * qr - si * qi : sr * qi + si * qr;
      } else {
        x = KIND == 0 ? (double)srow[i] : (double)srow[i] * (double)rrow[i];
      }
      const float dv = drow[i];
      pos += x * (double)dv;
      a.snap[p * d + i] = srow[i];
      a.mix[p * d + i] = -(double)dv;
    }
    const float xt = to_tf32((float)x);
    *reinterpret_cast<float*>(tile + cm_offset(rr, i, dp)) = xt;
    *reinterpret_cast<float*>(tslice + cm_offset(i, rt, 64)) = xt;
  }
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

// One warp per padded negative slot (chunk, j < kpad): the TF32 row in the
// core-matrix layout and, for j < k, the negative's contribution item.
__global__ void __launch_bounds__(256) shared_gather_kernel(BatchArgs a) {
  const uint64_t slot = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t d = a.dim, dp = a.dpad, k = a.k, kp = a.kpad;
  if (slot >= a.nch * kp) return;
  const uint64_t c = slot / kp;
  const uint32_t j = (uint32_t)(slot - c * kp);
  unsigned char* blk = reinterpret_cast<unsigned char*>(a.sh_B) + (slot >> 6) * 64ull * dp * 4;
  unsigned char* tblk = reinterpret_cast<unsigned char*>(a.sh_BT) + (slot >> 6) * 64ull * dp * 4;
  const uint32_t rr = (uint32_t)(slot & 63);
  if (j >= k) {
    for (uint32_t i = lane; i < dp; i += 32) {
      *reinterpret_cast<float*>(blk + cm_offset(rr, i, dp)) = 0.f;
      *reinterpret_cast<float*>(tblk + cm_offset(i, rr, 64)) = 0.f;
    }
    return;
  }
  const uint32_t id = a.negs[c * k + j];
  const float* row = a.theta + (size_t)id * d;
  for (uint32_t i = lane; i < dp; i += 32) {
    const float v = i < d ? to_tf32(row[i]) : 0.f;
    *reinterpret_cast<float*>(blk + cm_offset(rr, i, dp)) = v;
    *reinterpret_cast<float*>(tblk + cm_offset(i, rr, 64)) = v;
  }
  if (lane == 0) {
    const uint64_t item = 2 * a.P + c * k + j;
    a.node_keys[item] = pool_index(a, id);
    a.node_vals[item] = (uint32_t)((c * kp + j) << 2) | 1u;  // slot 1: shared negative
  }
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

// SG1: per tile, S = IR1 N^T in 64-negative blocks; online max / sum of exp
// per row -> M_p, 1/Z_p and loss_p = -(pos_p - (M_p + log Z_p)) (train.cpp:274).
__global__ void __launch_bounds__(kThreads, 1) sg1_stats_kernel(BatchArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t dp = a.dpad, k = a.k, kp = a.kpad;
  const uint32_t tile_bytes = 128 * dp * 4, blk_bytes = kNegBlk * dp * 4;
  unsigned char* sA = smem;
  unsigned char* sN = smem + tile_bytes;  // two blocks
  __shared__ uint64_t bars[4];            // 0: A, 1-2: N buffers, 3: MMA
  __shared__ uint32_t tbase_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const TileGeom g = tile_geom(a, blockIdx.x);
  if (warp == 0) tmem_alloc(&tbase_s, 64);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) bar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  const uint32_t nblk = kp / kNegBlk;
  const unsigned char* gA = reinterpret_cast<const unsigned char*>(a.sh_A) + g.row0 * dp * 4;
  const unsigned char* gN =
      reinterpret_cast<const unsigned char*>(a.sh_B) + g.c * (uint64_t)kp * dp * 4;
  if (tid == 0) {
    bar_expect(bars, tile_bytes);
    bulk_load(sA, gA, tile_bytes, bars);
    for (uint32_t b = 0; b < 2 && b < nblk; ++b) {
      bar_expect(bars + 1 + b, blk_bytes);
      bulk_load(sN + b * blk_bytes, gN + (uint64_t)b * blk_bytes, blk_bytes, bars + 1 + b);
    }
  }
  const uint32_t idesc = instr_desc(128, kNegBlk, false, false);
  const uint32_t kcore = (dp / 4) * 128;  // SBO: next 8-row group
  float m = -INFINITY, z = 0.f;
  const uint32_t row = tid;
  for (uint32_t nb = 0; nb < nblk; ++nb) {
    const uint32_t buf = nb & 1;
    if (tid == 0) {
      if (nb == 0) bar_wait(bars, 0);
      bar_wait(bars + 1 + buf, (nb >> 1) & 1);
      tc_fence_after();
      const uint32_t a0 = saddr(sA), b0 = saddr(sN + buf * blk_bytes);
      for (uint32_t ks = 0; ks < dp / 8; ++ks)
        mma_tf32(tbase, smem_desc(a0 + ks * 256, 128, kcore), smem_desc(b0 + ks * 256, 128, kcore),
                 idesc, ks > 0);
      mma_commit(bars + 3);
    }
    bar_wait(bars + 3, nb & 1);
    tc_fence_after();
    if (tid == 0 && nb + 2 < nblk) {  // the MMA is done with this buffer
      bar_expect(bars + 1 + buf, blk_bytes);
      bulk_load(sN + buf * blk_bytes, gN + (uint64_t)(nb + 2) * blk_bytes, blk_bytes,
                bars + 1 + buf);
    }
    float v[kNegBlk];
    const uint32_t lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
#pragma unroll
    for (int q = 0; q < kNegBlk; q += 16) tmem_ld16(lane_addr + q, v + q);
    float bm = -INFINITY;
#pragma unroll
    for (int q = 0; q < kNegBlk; ++q)
      if (nb * kNegBlk + q < k) bm = fmaxf(bm, v[q]);
    const float mn = fmaxf(m, bm);
    float zs = 0.f;
#pragma unroll
    for (int q = 0; q < kNegBlk; ++q)
      if (nb * kNegBlk + q < k) zs += __expf(v[q] - mn);
    z = (m == -INFINITY ? 0.f : z * __expf(m - mn)) + zs;
    m = mn;
    tc_fence_before();
    __syncthreads();
  }
  if (row < g.valid) {
    const uint64_t tr = g.row0 + row;
    a.sh_rowmax[tr] = m;
    a.sh_rowinv[tr] = 1.f / z;
    const uint64_t p = g.c * a.chunk + (tr - g.c * (uint64_t)a.tpc * 128);
    a.loss[p] = -(a.sh_pos[p] - ((double)m + log((double)z)));
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tbase, 64);
}

// SG2: per tile, mix += W N with W = exp(S - M) / Z recomputed block by block.
// TMEM: mix accumulator in columns [0, dpad), S in [scol, scol + 64).
__global__ void __launch_bounds__(kThreads, 1) sg2_mix_kernel(BatchArgs a, uint32_t tcols,
                                                              uint32_t scol) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t dp = a.dpad, k = a.k, kp = a.kpad, d = a.dim;
  const uint32_t tile_bytes = 128 * dp * 4, blk_bytes = kNegBlk * dp * 4;
  unsigned char* sA = smem;
  unsigned char* sN = smem + tile_bytes;            // two blocks: N (64 x dpad) then N^T
  unsigned char* sW = sN + 4 * blk_bytes;           // 128 x 64 f32, core-matrix layout
  __shared__ uint64_t bars[5];  // 0: A, 1-2: N buffers, 3: S MMA, 4: mix MMA
  __shared__ uint32_t tbase_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const TileGeom g = tile_geom(a, blockIdx.x);
  if (warp == 0) tmem_alloc(&tbase_s, tcols);
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) bar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  const uint32_t nblk = kp / kNegBlk;
  const unsigned char* gA = reinterpret_cast<const unsigned char*>(a.sh_A) + g.row0 * dp * 4;
  const unsigned char* gN =
      reinterpret_cast<const unsigned char*>(a.sh_B) + g.c * (uint64_t)kp * dp * 4;
  const unsigned char* gNT =
      reinterpret_cast<const unsigned char*>(a.sh_BT) + g.c * (uint64_t)kp * dp * 4;
  // buffer b: N block at sN + 2b blk, N^T block right after it
  auto load_blk = [&](uint32_t nb, uint32_t b) {
    bar_expect(bars + 1 + b, 2 * blk_bytes);
    bulk_load(sN + 2 * b * blk_bytes, gN + (uint64_t)nb * blk_bytes, blk_bytes, bars + 1 + b);
    bulk_load(sN + (2 * b + 1) * blk_bytes, gNT + (uint64_t)nb * blk_bytes, blk_bytes,
              bars + 1 + b);
  };
  if (tid == 0) {
    bar_expect(bars, tile_bytes);
    bulk_load(sA, gA, tile_bytes, bars);
    for (uint32_t b = 0; b < 2 && b < nblk; ++b) load_blk(b, b);
  }
  const uint32_t row = tid;
  const bool valid = row < g.valid;
  const float rm = valid ? a.sh_rowmax[g.row0 + row] : 0.f;
  const float ri = valid ? a.sh_rowinv[g.row0 + row] : 0.f;
  const uint32_t kcore = (dp / 4) * 128;
  const uint32_t id_s = instr_desc(128, kNegBlk, false, false);
  const uint32_t id_m = instr_desc(128, dp, false, false);
  const uint32_t lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
  for (uint32_t nb = 0; nb < nblk; ++nb) {
    const uint32_t buf = nb & 1;
    if (tid == 0) {
      if (nb == 0) bar_wait(bars, 0);
      if (nb >= 1) {  // mix MMA of block nb-1 done: its N buffer is free
        bar_wait(bars + 4, (nb - 1) & 1);
        if (nb + 1 < nblk) load_blk(nb + 1, (nb + 1) & 1);
      }
      bar_wait(bars + 1 + buf, (nb >> 1) & 1);
      tc_fence_after();
      const uint32_t a0 = saddr(sA), b0 = saddr(sN + 2 * buf * blk_bytes);
      for (uint32_t ks = 0; ks < dp / 8; ++ks)
        mma_tf32(tbase + scol, smem_desc(a0 + ks * 256, 128, kcore),
                 smem_desc(b0 + ks * 256, 128, kcore), id_s, ks > 0);
      mma_commit(bars + 3);
    }
    bar_wait(bars + 3, nb & 1);
    tc_fence_after();
    float v[kNegBlk];
#pragma unroll
    for (int q = 0; q < kNegBlk; q += 16) tmem_ld16(lane_addr + scol + q, v + q);
    if (nb >= 1) bar_wait(bars + 4, (nb - 1) & 1);  // W buffer free again
#pragma unroll
    for (int q = 0; q < kNegBlk; q += 4) {
      float4 w;
      const uint32_t j = nb * kNegBlk + q;
      w.x = (valid && j + 0 < k) ? __expf(v[q + 0] - rm) * ri : 0.f;
      w.y = (valid && j + 1 < k) ? __expf(v[q + 1] - rm) * ri : 0.f;
      w.z = (valid && j + 2 < k) ? __expf(v[q + 2] - rm) * ri : 0.f;
      w.w = (valid && j + 3 < k) ? __expf(v[q + 3] - rm) * ri : 0.f;
      w.x = to_tf32(w.x), w.y = to_tf32(w.y), w.z = to_tf32(w.z), w.w = to_tf32(w.w);
      *reinterpret_cast<float4*>(sW + cm_offset(row, q, kNegBlk)) = w;
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t w0 = saddr(sW), t0 = saddr(sN + (2 * buf + 1) * blk_bytes);
      // A = W (128 x 64 negatives), B = N^T (dpad x 64 negatives), both K-major
      for (uint32_t ks = 0; ks < kNegBlk / 8; ++ks)
        mma_tf32(tbase, smem_desc(w0 + ks * 256, 128, (kNegBlk / 4) * 128),
                 smem_desc(t0 + ks * 256, 128, (kNegBlk / 4) * 128), id_m, (nb | ks) != 0);
      mma_commit(bars + 4);
    }
  }
  bar_wait(bars + 4, (nblk - 1) & 1);
  tc_fence_after();
  {
    const uint64_t tr = g.row0 + row;
    const uint64_t p = g.c * a.chunk + (tr - g.c * (uint64_t)a.tpc * 128);
    double* mx = a.mix + p * d;
    for (uint32_t q = 0; q < dp; q += 16) {  // collective loads: every lane, every step
      float v[16];
      tmem_ld16(lane_addr + q, v);
      if (valid) {
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (q + e < d) mx[q + e] += (double)v[e];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tbase, tcols);
}

// SG3: per (chunk, 128 negatives): G = W^T IR1 over the chunk's positives in
// 64-positive slices; S^T = N IR1^T is recomputed per slice (M = the 128
// negatives, N = 64 positives).  TMEM: G in [0, dpad), S^T in [scol, +64).
__global__ void __launch_bounds__(kThreads, 1) sg3_grad_kernel(BatchArgs a, uint32_t tcols,
                                                               uint32_t scol) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t dp = a.dpad, k = a.k, kp = a.kpad, d = a.dim;
  const uint32_t nblk_bytes = 128 * dp * 4, sl_bytes = kPosSlice * dp * 4;
  unsigned char* sN = smem;                 // 128 negatives x dpad
  unsigned char* sA = smem + nblk_bytes;    // two buffers: IR1 slice (64 x dpad), then IR1^T
  unsigned char* sW = sA + 4 * sl_bytes;    // W^T: 128 negatives x 64 positives
  __shared__ uint64_t bars[5];  // 0: N, 1-2: slices, 3: S MMA, 4: G MMA
  __shared__ uint32_t tbase_s;
  __shared__ float s_m[kPosSlice], s_i[kPosSlice];
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t nbpc = kp / 128;  // negative blocks per chunk
  const uint64_t c = blockIdx.x / nbpc;
  const uint32_t n0 = (blockIdx.x - c * nbpc) * 128;
  const uint64_t left = a.P - c * a.chunk;
  const uint64_t chunk_rows = left < a.chunk ? left : a.chunk;
  const uint32_t nsl = (uint32_t)((chunk_rows + kPosSlice - 1) / kPosSlice);
  if (warp == 0) tmem_alloc(&tbase_s, tcols);
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) bar_init(bars + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;
  const uint64_t crow0 = c * (uint64_t)a.tpc * 128;  // the chunk's first padded row
  const unsigned char* gA = reinterpret_cast<const unsigned char*>(a.sh_A) + crow0 * dp * 4;
  const unsigned char* gAT = reinterpret_cast<const unsigned char*>(a.sh_AT) + crow0 * dp * 4;
  const unsigned char* gN =
      reinterpret_cast<const unsigned char*>(a.sh_B) + (c * (uint64_t)kp + n0) * dp * 4;
  auto load_slice = [&](uint32_t s, uint32_t b) {
    bar_expect(bars + 1 + b, 2 * sl_bytes);
    bulk_load(sA + 2 * b * sl_bytes, gA + (uint64_t)s * sl_bytes, sl_bytes, bars + 1 + b);
    bulk_load(sA + (2 * b + 1) * sl_bytes, gAT + (uint64_t)s * sl_bytes, sl_bytes, bars + 1 + b);
  };
  if (tid == 0) {
    bar_expect(bars, nblk_bytes);
    bulk_load(sN, gN, nblk_bytes, bars);
    for (uint32_t s = 0; s < 2 && s < nsl; ++s) load_slice(s, s);
  }
  const uint32_t row = tid;  // negative n0 + row
  const bool nvalid = n0 + row < k;
  const uint32_t kcore = (dp / 4) * 128;
  const uint32_t id_s = instr_desc(128, kPosSlice, false, false);
  const uint32_t id_g = instr_desc(128, dp, false, false);
  const uint32_t lane_addr = tbase + ((uint32_t)(warp * 32) << 16);
  for (uint32_t s = 0; s < nsl; ++s) {
    const uint32_t buf = s & 1;
    if (tid < kPosSlice) {  // row statistics of this slice's positives
      const uint64_t q = (uint64_t)s * kPosSlice + tid;
      s_m[tid] = q < chunk_rows ? a.sh_rowmax[crow0 + q] : 0.f;
      s_i[tid] = q < chunk_rows ? a.sh_rowinv[crow0 + q] : 0.f;
    }
    if (tid == 0) {
      if (s == 0) bar_wait(bars, 0);
      if (s >= 1) {
        bar_wait(bars + 4, (s - 1) & 1);
        if (s + 1 < nsl) load_slice(s + 1, (s + 1) & 1);
      }
      bar_wait(bars + 1 + buf, (s >> 1) & 1);
      tc_fence_after();
      const uint32_t a0 = saddr(sN), b0 = saddr(sA + 2 * buf * sl_bytes);
      for (uint32_t ks = 0; ks < dp / 8; ++ks)
        mma_tf32(tbase + scol, smem_desc(a0 + ks * 256, 128, kcore),
                 smem_desc(b0 + ks * 256, 128, kcore), id_s, ks > 0);
      mma_commit(bars + 3);
    }
    bar_wait(bars + 3, s & 1);
    tc_fence_after();
    __syncthreads();  // s_m / s_i visible
    float v[kPosSlice];
#pragma unroll
    for (int q = 0; q < kPosSlice; q += 16) tmem_ld16(lane_addr + scol + q, v + q);
    if (s >= 1) bar_wait(bars + 4, (s - 1) & 1);
#pragma unroll
    for (int q = 0; q < kPosSlice; q += 4) {
      float w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t pq = (uint64_t)s * kPosSlice + q + e;
        w[e] = (nvalid && pq < chunk_rows) ? to_tf32(__expf(v[q + e] - s_m[q + e]) * s_i[q + e])
                                           : 0.f;
      }
      *reinterpret_cast<float4*>(sW + cm_offset(row, q, kPosSlice)) =
          make_float4(w[0], w[1], w[2], w[3]);
    }
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t w0 = saddr(sW), t0 = saddr(sA + (2 * buf + 1) * sl_bytes);
      // A = W^T (128 negatives x 64 positives), B = IR1^T (dpad x 64 positives)
      for (uint32_t ks = 0; ks < kPosSlice / 8; ++ks)
        mma_tf32(tbase, smem_desc(w0 + ks * 256, 128, (kPosSlice / 4) * 128),
                 smem_desc(t0 + ks * 256, 128, (kPosSlice / 4) * 128), id_g, (s | ks) != 0);
      mma_commit(bars + 4);
    }
  }
  bar_wait(bars + 4, (nsl - 1) & 1);
  tc_fence_after();
  float* gout = a.sh_G + (c * (uint64_t)kp + n0 + row) * d;
  for (uint32_t q = 0; q < dp; q += 16) {
    float v[16];
    tmem_ld16(lane_addr + q, v);
    if (nvalid) {
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (q + e < d) gout[q + e] = v[e];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free(tbase, tcols);
}

uint32_t pow2_cols(uint32_t n) {
  uint32_t c = 32;
  while (c < n) c <<= 1;
  return c;
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  LGD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace

SharedShape shared_shape(uint32_t dim, uint32_t k, uint32_t chunk, uint64_t P) {
  SharedShape s{};
  s.dpad = (dim + 15) & ~15u;
  s.kpad = (k + 127) & ~127u;
  s.tpc = (chunk + 127) / 128;
  s.nch = chunk ? (P + chunk - 1) / chunk : 0;
  return s;
}

size_t shared_smem_bytes(uint32_t dpad) {
  const size_t t = 128ull * dpad * 4, b = (size_t)kNegBlk * dpad * 4;
  const size_t sg2 = t + 4 * b + 128 * kNegBlk * 4;
  const size_t sg3 = t + 4 * (size_t)kPosSlice * dpad * 4 + 128 * kPosSlice * 4;
  return sg2 > sg3 ? sg2 : sg3;
}

void launch_shared_scores(const BatchArgs& a, cudaStream_t st) {
  const uint64_t rows = a.nch * (uint64_t)a.tpc * 128;
  switch (a.kind) {
    case 0:
      shared_prep_kernel<0><<<ceil_div(rows * 32, 256), 256, 0, st>>>(a);
      break;
    case 1:
      shared_prep_kernel<1><<<ceil_div(rows * 32, 256), 256, 0, st>>>(a);
      break;
    default:
      shared_prep_kernel<2><<<ceil_div(rows * 32, 256), 256, 0, st>>>(a);
      break;
  }
  LGD_LAUNCH_CHECK();
  shared_gather_kernel<<<ceil_div(a.nch * (uint64_t)a.kpad * 32, 256), 256, 0, st>>>(a);
  LGD_LAUNCH_CHECK();
  const uint32_t dp = a.dpad;
  const size_t t = 128ull * dp * 4, b = (size_t)kNegBlk * dp * 4;
  const size_t sm1 = t + 2 * b;
  const size_t sm2 = t + 4 * b + 128 * kNegBlk * 4;
  const size_t sm3 = t + 4 * (size_t)kPosSlice * dp * 4 + 128 * kPosSlice * 4;
  static size_t set1 = 0, set2 = 0, set3 = 0;  // attributes only grow
  if (sm1 > set1) set_smem(sg1_stats_kernel, set1 = sm1);
  if (sm2 > set2) set_smem(sg2_mix_kernel, set2 = sm2);
  if (sm3 > set3) set_smem(sg3_grad_kernel, set3 = sm3);
  const unsigned tiles = (unsigned)(a.nch * a.tpc);
  const uint32_t scol = (dp + 31) & ~31u;
  const uint32_t tcols = pow2_cols(scol + 64);
  sg1_stats_kernel<<<tiles, kThreads, sm1, st>>>(a);
  LGD_LAUNCH_CHECK();
  sg2_mix_kernel<<<tiles, kThreads, sm2, st>>>(a, tcols, scol);
  LGD_LAUNCH_CHECK();
  sg3_grad_kernel<<<(unsigned)(a.nch * (a.kpad / 128)), kThreads, sm3, st>>>(a, tcols, scol);
  LGD_LAUNCH_CHECK();
}

}  // namespace lgd
