// context.hpp -- the trainer context behind the C ABI (lgd_context) and its
// host epoch driver; context.cu holds the C entry points, rounds.cu the
// multi-GPU partition-round runner.
//
// The driver is the real-train branch of run_epoch (pipeline.cpp:273-322)
// with every partition resident in HBM: the SSD tier, NVMe simulation and
// state-boundary swaps of the reference become a change of the sampling
// pool (the partitions of the current plan state), exactly the reference's
// own in-memory restatement (test_pipeline.cpp:227-269).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/legend_b200.h"
#include "abi.hpp"
#include "common.cuh"
#include "evaluate.cuh"
#include "internal.hpp"
#include "planner.hpp"
#include "rng.cuh"
#include "train.cuh"

using namespace lgd;

namespace lgd {

struct RoundRunner;  // rounds.cu
void destroy_round_runner(RoundRunner* r);
struct RunnerDeleter {
  void operator()(RoundRunner* r) const { destroy_round_runner(r); }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    LGD_CUDA(cudaGetDevice(&prev));
    if (prev != dev) LGD_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

constexpr int kProfRing = 256;

}  // namespace lgd

struct lgd_context {
  int device = 0;
  int kind = 0;
  uint32_t dim = 0;
  lgd_train_options opt{};
  cudaStream_t stream = nullptr;
  int sm_count = 148;

  // graph
  uint64_t V = 0, R = 0, E = 0;
  DevBuf<uint32_t> edges;         // ingest order, E x 3
  DevBuf<uint32_t> edges_bucketed;  // bucket order (edge_order applied), E x 3
  bool partitioned = false;
  uint32_t n = 0;
  uint64_t stride = 0;
  std::vector<uint64_t> offsets;  // n*n + 1
  bool planned = false;
  IterationPlan plan;

  // tables
  DevBuf<float> theta, state, rel_theta, rel_state;
  bool tables_ready = false;

  // per-bucket scratch
  uint64_t bucket_cap = 0;
  DevBuf<uint32_t> H, perm, shuffled, negs;
  DevBuf<uint32_t> sh_keys_in, sh_vals_in, sh_keys_out, sh_vals_out, sh_ptr, sh_G;
  DevBuf<unsigned char> sh_temp;
  DevBuf<uint64_t> pos;
  DevBuf<unsigned long long> reject;

  // per-batch scratch
  uint64_t batch_cap = 0;  // positives
  uint32_t k_cap = 0;
  DevBuf<double> w, mix, ir1, loss, part_first, part_last;
  DevBuf<float> snap;
  // shared-negative chunks (shared.cu)
  DevBuf<float> sn_A, sn_AT, sn_B, sn_BT, sn_D, sn_rowc, sn_G;
  DevBuf<double> sn_pos;
  DevBuf<uint32_t> node_keys, node_vals, rel_keys, iota, skeys, svals;
  // bucket-level presort (presort_bucket): keys / payloads and their
  // double-buffer partners; the batches of the bucket read runs of the result
  DevBuf<uint32_t> bk_keys[2], bk_vals[2];
  DevBuf<unsigned char> bk_temp;
  bool presort = true;  // LGD_PRESORT=0 turns it off (per-batch sorts)
  // K4 v2 (train.cu: segment_rows) over a segment list; LGD_K4=1 selects the
  // chunked pass 1 / pass 2 kernels instead (A/B)
  bool seg_rows = true;
  // K4 v2 kernel: 0 segment_heads, 1 warp-specialised (LGD_K4=3), 2 flattened (LGD_K4=4)
  int k4_variant = 0;
  DevBuf<uint32_t> long_head, long_end, long_chunk_base, long_first, nlong;
  DevBuf<double> rel64;  // FP64 relation rows for K4 (K3 writes them; R <= kRel64Max)
  static constexpr uint64_t kRel64Max = 256;
  DevBuf<unsigned char> seg_temp;
  bool bucket_segs = false;  // the current bucket's long-segment list is built
  cudaEvent_t ev_long = nullptr, ev_long_done = nullptr;
  struct Presorted {
    const uint32_t* keys = nullptr;
    const uint32_t* vals = nullptr;
    uint32_t mask = 0;
    int rel_bits = 0;  // payload layout of the whole bucket
    uint64_t items = 0;
  } bk;
  // Bucket-prep overlap (LGD_OVERLAP_PREP=1, opt-in): the next bucket's
  // shuffle / sample / presort / segment list run on prep_stream into a
  // second set of the per-bucket buffers while the batches of the current
  // bucket run on `stream`.  The members above always hold the set being
  // enqueued; swap_sets() exchanges them with `alt`.  Only the outputs are
  // doubled: the prep-only scratch (H, perm, sh_*, pos, reject) is used by
  // one prep at a time, all on prep_stream.
  struct BucketSet {
    DevBuf<uint32_t> shuffled, negs, keys[2], vals[2];
    DevBuf<uint32_t> long_head, long_end, long_chunk_base, long_first, nlong;
    DevBuf<unsigned char> bk_temp, seg_temp;
    Presorted bk;
    bool segs = false;
  } alt;
  // measured on TW: no gain (plan 87.5M vs 87.7M edges/s serial; rounds
  // 89.9M vs 90.4M: the prep's sorts run in K4's gaps and stretch K4 by the
  // SMs they hold), so the serial prep stays the default
  bool overlap_prep = false;
  int set_id = 0;  // which of the two physical sets the members hold
  cudaStream_t prep_stream = nullptr;
  cudaEvent_t ev_prepped[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
  void swap_sets() {
    shuffled.swap(alt.shuffled);
    negs.swap(alt.negs);
    for (int i = 0; i < 2; ++i) {
      bk_keys[i].swap(alt.keys[i]);
      bk_vals[i].swap(alt.vals[i]);
    }
    long_head.swap(alt.long_head);
    long_end.swap(alt.long_end);
    long_chunk_base.swap(alt.long_chunk_base);
    long_first.swap(alt.long_first);
    nlong.swap(alt.nlong);
    bk_temp.swap(alt.bk_temp);
    seg_temp.swap(alt.seg_temp);
    std::swap(bk, alt.bk);
    std::swap(bucket_segs, alt.segs);
    set_id ^= 1;
  }
  // the second set sized like the first (after reserve_for)
  void reserve_alt() {
    alt.shuffled.reserve(shuffled.n);
    alt.negs.reserve(negs.n);
    for (int i = 0; i < 2; ++i) {
      alt.keys[i].reserve(bk_keys[i].n);
      alt.vals[i].reserve(bk_vals[i].n);
    }
    alt.long_head.reserve(long_head.n);
    alt.long_end.reserve(long_end.n);
    alt.long_chunk_base.reserve(long_chunk_base.n);
    alt.long_first.reserve(long_first.n);
    alt.nlong.reserve(nlong.n);
    alt.bk_temp.reserve(bk_temp.n);
    alt.seg_temp.reserve(seg_temp.n);
  }
  DevBuf<uint8_t> chunk_flags;
  DevBuf<uint32_t> span_list;
  DevBuf<unsigned int> span_count;
  DevBuf<unsigned char> sort_temp;
  DevBuf<unsigned long long> counters;
  DevBuf<double> batch_losses;
  DevBuf<uint32_t> op_edges, op_negs;  // operator-level uploads
  // relation pass on the side stream (train.cuh: BatchArgs::side)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_scored = nullptr, ev_rel = nullptr;
  DevBuf<uint32_t> r_skeys, r_svals, r_span_list;
  DevBuf<unsigned char> r_sort_temp;
  DevBuf<double> r_part_first, r_part_last, r_grad;
  DevBuf<uint8_t> r_chunk_flags, r_touched;
  DevBuf<unsigned int> r_span_count;

  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> prof_events;  // kProfRing x 5
  std::vector<int> prof_pending;
  int prof_head = 0;
  lgd_kernel_stats kstats[LGD_KSTAT_COUNT]{};
  cudaEvent_t ev_begin = nullptr, ev_end = nullptr;
  cudaStream_t copy_stream = nullptr;
  // asynchronous partition write-back (lgd_store_partition_async): D2H copies
  // on their own stream, ordered after the training stream's work so far;
  // the next call that writes the tables first orders itself after them
  cudaStream_t store_stream = nullptr;
  cudaEvent_t ev_store_src = nullptr, ev_store_done = nullptr;
  bool stores_pending = false;
  cudaEvent_t copy_done[2] = {nullptr, nullptr}, stage_free[2] = {nullptr, nullptr};
  DevBuf<uint32_t> staging[2];
  uint64_t launches = 0;
  size_t l2_persist = 0, l2_window_max = 0;  // L2 set-aside for the snapshot rows
  // optional host copy of the bucket-ordered edges (lgd_set_host_edges): the
  // bucket lists and rounds then stream every bucket H2D instead of reading
  // the device copy
  const uint32_t* host_edges = nullptr;
  uint64_t round_h2d = 0;
  double score_bytes_total = 0.0;  // algorithmic score-phase bytes since the call began

  // multi-GPU partition-round runner (rounds.cu; lgd_comm_init)
  std::unique_ptr<RoundRunner, RunnerDeleter> runner;

  ~lgd_context() {
    cudaSetDevice(device);
    runner.reset();  // peer mappings and events before the tables
    if (store_stream) cudaStreamSynchronize(store_stream);  // before the tables are freed
    if (store_stream) cudaStreamDestroy(store_stream);
    if (ev_store_src) cudaEventDestroy(ev_store_src);
    if (ev_store_done) cudaEventDestroy(ev_store_done);
    if (stream) cudaStreamDestroy(stream);
    for (auto e : prof_events) cudaEventDestroy(e);
    if (ev_begin) cudaEventDestroy(ev_begin);
    if (ev_end) cudaEventDestroy(ev_end);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (side_stream) cudaStreamDestroy(side_stream);
    if (ev_scored) cudaEventDestroy(ev_scored);
    if (ev_rel) cudaEventDestroy(ev_rel);
    if (ev_long) cudaEventDestroy(ev_long);
    if (ev_long_done) cudaEventDestroy(ev_long_done);
    for (auto e : {copy_done[0], copy_done[1], stage_free[0], stage_free[1], ev_prepped[0],
                   ev_prepped[1], ev_consumed[0], ev_consumed[1]})
      if (e) cudaEventDestroy(e);
    if (prep_stream) cudaStreamDestroy(prep_stream);
  }

  // Orders every later launch on `stream` (the only stream that writes the
  // tables) after the pending asynchronous write-backs.
  void fence_stores() {
    if (!stores_pending) return;
    LGD_CUDA(cudaStreamWaitEvent(stream, ev_store_done, 0));
    stores_pending = false;
  }
  // The same on the host, for writes that do not go through `stream`.
  void wait_stores() {
    if (store_stream) LGD_CUDA(cudaStreamSynchronize(store_stream));
    stores_pending = false;
  }

  bool typed() const { return kind != LGD_MODEL_DOT; }
  uint32_t k() const { return opt.negatives; }
  uint32_t chunk() const { return opt.shared_chunk; }
  // negative ids a batch of P positives draws: P k, or ceil(P / C) k shared
  uint64_t batch_negs(uint64_t P) const {
    return chunk() ? (P + chunk() - 1) / chunk() * k() : P * k();
  }
  // a bucket's draws: its batches' in order (pipeline.cpp:303-308)
  uint64_t bucket_negs(uint64_t m) const {
    const uint64_t B = opt.batch_size, full = m / B, rest = m - full * B;
    return full * batch_negs(B) + batch_negs(rest);
  }
  uint64_t batch_items(uint64_t P) const {  // node-gradient contributions
    return chunk() ? 2 * P + batch_negs(P) : P * (k() + 2);
  }

  uint64_t part_begin(uint32_t p) const { return stride * p; }
  uint64_t part_rows(uint32_t p) const {
    const uint64_t b = stride * p, e = std::min<uint64_t>(stride * (p + 1), V);
    return e > b ? e - b : 0;
  }

  void ensure_bucket(uint64_t m) {
    if (m <= bucket_cap) return;
    const uint64_t cap = m;
    H.reserve(cap);
    perm.reserve(cap);
    shuffled.reserve(cap * 3);
    negs.reserve(std::max<uint64_t>(bucket_negs(cap), 1));
    sh_keys_in.reserve(cap);
    sh_vals_in.reserve(cap);
    sh_keys_out.reserve(cap);
    sh_vals_out.reserve(cap);
    sh_ptr.reserve(cap);
    sh_G.reserve(cap);
    sh_temp.reserve(shuffle_sort_temp_bytes(cap));
    bucket_cap = cap;
  }

  void ensure_batch(uint64_t P) {
    const uint32_t kk = k();
    if (P <= batch_cap && kk <= k_cap) return;
    P = std::max(P, batch_cap);
    const uint64_t items = batch_items(P);
    if (chunk()) {
      const SharedShape sh = shared_shape(dim, kk, chunk(), P);
      const uint64_t rows = sh.nch * sh.tpc * 128;
      sn_A.reserve(rows * sh.dpad);
      sn_AT.reserve(rows * sh.dpad);
      sn_D.reserve(rows * dim + 4);  // + slack: SG2 copies whole 16-byte pieces
      sn_B.reserve(sh.nch * sh.kpad * sh.dpad);
      sn_BT.reserve(sh.nch * sh.kpad * sh.dpad);
      sn_rowc.reserve(rows);
      sn_G.reserve(sh.nch * sh.kpad * dim);
      sn_pos.reserve(P);
    } else {
      w.reserve(P * kk + P);  // + TransE's dst coefficients
    }
    mix.reserve(P * dim);
    if (use_ir1()) ir1.reserve(P * dim);  // K3 -> K4 IR1 rows
    snap.reserve(P * dim);
    loss.reserve(3 * P);  // K3's loss parts (loss_reduce takes the log)
    node_keys.reserve(items);
    node_vals.reserve(items);
    rel_keys.reserve(P);
    skeys.reserve(items);
    svals.reserve(items);
    const uint64_t chunks = (items + 31) / 32;
    // (K4 v2's long-segment chunk partials: at most 2 items / 32 rows)
    part_first.reserve((2 * chunks + 1) * dim);
    part_last.reserve(chunks * dim);
    chunk_flags.reserve(chunks);
    span_list.reserve(chunks);
    span_count.reserve(1);
    sort_temp.reserve(batch_sort_temp_bytes(items));
    if (iota.n < items) {
      iota.reserve(items);
      std::vector<uint32_t> h(items);
      for (uint64_t i = 0; i < items; ++i) h[i] = (uint32_t)i;
      LGD_CUDA(cudaMemcpy(iota.get(), h.data(), items * 4, cudaMemcpyHostToDevice));
    }
    if (typed()) {
      const uint64_t rchunks = (P + 31) / 32;
      r_skeys.reserve(P);
      r_svals.reserve(P);
      r_sort_temp.reserve(batch_sort_temp_bytes(P));
      r_part_first.reserve(rchunks * dim);
      r_part_last.reserve(rchunks * dim);
      r_chunk_flags.reserve(rchunks);
      r_span_list.reserve(rchunks);
      r_span_count.reserve(1);
      r_grad.reserve(std::max<uint64_t>(R, 1) * dim);
      r_touched.reserve(std::max<uint64_t>(R, 1));
    }
    if (seg_rows) ensure_segments(items, 1);
    batch_cap = P;
    k_cap = kk;
    pin_snapshot_in_l2();
  }

  // K3 stores IR1 rows for K4 only where K4 reads them: ComplEx / TransE
  // (k4_ir1), the exact path, vector-lane dims; LGD_K4_IR1=0 recombines the
  // snapshot instead (same bits; tests A/B the two).  The chunked K4 kernels
  // always read them.
  bool ir1_rows = true;
  bool use_ir1() const {
    return k4_ir1(kind) && !chunk() && k4_vec_width(kind, dim) != 0 && (ir1_rows || !seg_rows);
  }

  // segment-list scratch for up to `items` sorted contributions in `nb` batches
  void ensure_segments(uint64_t items, uint64_t nb) {
    long_head.reserve(items / 33 + 1);
    long_end.reserve(items / 33 + 1);
    long_chunk_base.reserve(items / 33 + 2);
    long_first.reserve(nb + 1);
    nlong.reserve(1);
    const size_t tb = long_list_temp_bytes(items);
    if (seg_temp.bytes() < tb) seg_temp.reserve(tb);
  }
  SegLists seg_lists() const {
    return SegLists{long_head.get(), long_end.get(), long_chunk_base.get(), long_first.get(),
                    nlong.get(), seg_temp.get(), seg_temp.bytes()};
  }

  // Every contribution of a positive reads its snapshot row (400 B at d = 100)
  // at a scattered time during K4 while the theta / state rows stream through
  // L2: a persisting access window keeps the snapshot on chip.
  void pin_snapshot_in_l2() {
    // (k4_ir1 models: K4 reads K3's f64 IR1 rows instead)
    const bool rows = use_ir1();
    void* base = rows ? (void*)ir1.get() : (void*)snap.get();
    const size_t bytes = rows ? ir1.bytes() : snap.bytes();
    if (!l2_persist || !base) return;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = base;
    v.accessPolicyWindow.num_bytes = std::min<size_t>(bytes, l2_window_max);
    v.accessPolicyWindow.hitRatio =
        (float)std::min(1.0, (double)l2_persist / (double)v.accessPolicyWindow.num_bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    LGD_CUDA(cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, &v));
  }

  BatchArgs batch_args(const uint32_t* bedges, const uint32_t* bnegs, uint64_t P,
                       double* loss_out, const Pool* pool = nullptr) const {
    BatchArgs a{};
    a.kind = kind;
    a.dim = dim;
    a.k = k();
    a.P = P;
    a.num_nodes = V;
    a.num_rels = R;
    a.edges = bedges;
    a.negs = bnegs;
    a.theta = theta.get();
    a.state = state.get();
    a.rel_theta = rel_theta.get();
    a.rel64 = nullptr;
    if (seg_rows && typed() && R && R <= kRel64Max && !chunk()) {
      const_cast<DevBuf<double>&>(rel64).reserve(R * dim);
      a.rel64 = rel64.get();
    }
    a.rel_state = rel_state.get();
    a.lr = opt.learning_rate;
    a.eps = opt.adagrad_epsilon;
    a.w = w.get();
    a.mix = mix.get();
    a.ir1 = use_ir1() ? ir1.get() : nullptr;
    a.snap = snap.get();
    a.loss = loss.get();
    a.loss_parts = 0;  // run_batch turns them on where K3 writes them
    a.node_keys = node_keys.get();
    a.node_vals = node_vals.get();
    a.slot_bits = bits_for(a.k + 1);
    if ((P << a.slot_bits) >> 32) throw std::invalid_argument("batch too large for 32-bit payloads");
    // the relation id rides in the payload when it fits: K4 then needs no
    // dependent rel_keys[p] load per contribution
    a.rel_bits = 0;
    if (typed() && R && !chunk()) {
      const int rb = bits_for(R - 1);
      if (bits_for(P ? P - 1 : 0) + a.slot_bits + rb <= 32) a.rel_bits = rb;
    }
    a.rel_keys = rel_keys.get();
    a.presorted = 0;
    a.key_mask = 0xffffffffu;
    a.iota = iota.get();
    a.skeys = skeys.get();
    a.svals = svals.get();
    a.sort_temp = sort_temp.get();
    a.sort_temp_bytes = sort_temp.bytes();
    a.part_first = part_first.get();
    a.part_last = part_last.get();
    a.chunk_flags = chunk_flags.get();
    a.span_list = span_list.get();
    a.span_count = span_count.get();
    a.counters = counters.get();
    a.batch_loss_out = loss_out;
    a.pool_first[0] = 0;
    a.pool_end[0] = V;
    a.pool_n = 1;
    a.node_key_bits = bits_for(V ? V - 1 : 0);
    if (pool) {  // keys are indices into the resident pool of the plan state
      for (int i = 0; i < 3; ++i) {
        a.pool_first[i] = pool->first[i];
        a.pool_end[i] = pool->end_index[i];
      }
      a.pool_n = pool->n;
      a.node_key_bits = bits_for(pool->end_index[pool->n - 1] - 1);
    }
    a.rel_key_bits = bits_for(R ? R - 1 : 0);
    a.sm_count = sm_count;
    a.gc = nullptr;
    a.k4_ws = k4_variant;
    a.seg_mode = seg_rows ? 2 : 0;  // run_batch switches to the bucket's list
    a.long_head = long_head.get();
    a.long_end = long_end.get();
    a.long_chunk_base = long_chunk_base.get();
    a.long_first = long_first.get();
    a.seg_lists = seg_lists();
    a.ev_long = ev_long;
    a.ev_long_done = ev_long_done;
    if (typed() && R && side_stream && r_grad.get()) {  // overlapped relation pass
      a.side = side_stream;
      a.ev_scored = ev_scored;
      a.ev_rel = ev_rel;
      a.num_rels = R;
      a.rel_skeys = r_skeys.get();
      a.rel_svals = r_svals.get();
      a.rel_sort_temp = r_sort_temp.get();
      a.rel_sort_temp_bytes = r_sort_temp.bytes();
      a.rel_part_first = r_part_first.get();
      a.rel_part_last = r_part_last.get();
      a.rel_chunk_flags = r_chunk_flags.get();
      a.rel_span_list = r_span_list.get();
      a.rel_span_count = r_span_count.get();
      a.rel_grad = r_grad.get();
      a.rel_touched = r_touched.get();
    } else if (!typed() && side_stream && !chunk()) {  // Dot: the loss reduction only
      a.side = side_stream;
      a.ev_scored = ev_scored;
      a.ev_rel = ev_rel;
    }
    if (chunk()) {
      const SharedShape sh = shared_shape(dim, a.k, chunk(), P);
      a.chunk = chunk();
      a.dpad = sh.dpad;
      a.kpad = sh.kpad;
      a.tpc = sh.tpc;
      a.nch = sh.nch;
      a.sh_A = sn_A.get();
      a.sh_B = sn_B.get();
      a.sh_AT = sn_AT.get();
      a.sh_BT = sn_BT.get();
      a.sh_rowc = sn_rowc.get();
      a.sh_D = sn_D.get();
      a.sh_pos = sn_pos.get();
      a.sh_G = sn_G.get();
    }
    return a;
  }

  // Shared-negative chunks: dot-product scores (the tensor-core contraction),
  // vector-lane dims (d % 4 == 0, ComplEx h even) up to 128.
  void check_shared() const {
    if (!chunk()) return;
    if (kind == LGD_MODEL_TRANSE)
      throw std::invalid_argument("shared negatives need a dot-product score (not TransE)");
    const bool vec = kind == LGD_MODEL_COMPLEX ? (dim / 2) % 2 == 0 : dim % 4 == 0;
    if (!vec || dim > 128)
      throw std::invalid_argument("shared negatives need dim % 4 == 0 (ComplEx: dim % 4) and dim <= 128");
  }

  uint64_t batch_launches(int node_bits = -1) const {
    if (chunk()) {  // prep, gather, SG1-3, loss, node sort, pass 1/2 (+ relation path)
      const int nb = node_bits >= 0 ? node_bits : bits_for(V ? V - 1 : 0);
      const int rb = bits_for(R ? R - 1 : 0);
      uint64_t c = 6 + 2 + 2 + (nb + 7) / 8;
      if (typed()) c += 2 + 2 + (rb + 7) / 8;
      return c;
    }
    // K3 + loss reduce + pass1 + pass2 (+ relation pass1/2) + radix sorts
    // (upsweep histogram + scan + one onesweep pass per 8 key bits)
    const int nb = node_bits >= 0 ? node_bits : bits_for(V ? V - 1 : 0);
    const int rb = bits_for(R ? R - 1 : 0);
    uint64_t c = 4 + 2 + (nb + 7) / 8;
    if (typed()) c += 2 + 2 + (rb + 7) / 8;
    return c;
  }

  // Profiling ring: slot = 5 events; a batch slot times 4 phases (score,
  // sort, update, relations), a bucket slot 2 (shuffle, sample).  Slots are
  // drained lazily (only when the ring wraps), so no host synchronisation
  // lands inside a timed region.
  int prof_slot(int kind) {
    const int slot = prof_head;
    prof_head = (prof_head + 1) % kProfRing;
    if (prof_pending[slot]) prof_drain(slot);
    prof_pending[slot] = kind;
    return slot;
  }
  cudaEvent_t* prof_ev(int slot) { return prof_events.data() + slot * 5; }

  void prof_drain(int slot) {
    cudaEvent_t* e = prof_ev(slot);
    const int kind = prof_pending[slot];
    const int nint = kind == 1 ? 4 : 3;
    LGD_CUDA(cudaEventSynchronize(e[nint]));
    const int batch_cls[4] = {LGD_KSTAT_SCORE, LGD_KSTAT_SORT, LGD_KSTAT_UPDATE, LGD_KSTAT_REL};
    const int bucket_cls[3] = {LGD_KSTAT_SHUFFLE, LGD_KSTAT_SAMPLE, LGD_KSTAT_SORT};
    for (int i = 0; i < nint; ++i) {
      const int cls = kind == 1 ? batch_cls[i] : bucket_cls[i];
      if (cls == LGD_KSTAT_REL && !typed()) continue;
      float ms = 0;
      LGD_CUDA(cudaEventElapsedTime(&ms, e[i], e[i + 1]));
      kstats[cls].launches += 1;
      kstats[cls].total_ms += ms;
    }
    prof_pending[slot] = 0;
  }

  void prof_flush() {
    if (prof_pending.empty()) return;
    for (int s = 0; s < kProfRing; ++s)
      if (prof_pending[s]) prof_drain(s);
  }

  void run_batch(const uint32_t* bedges, const uint32_t* bnegs, uint64_t P, double* loss_out,
                 const Pool* pool = nullptr, double* rel_grad_out = nullptr,
                 uint8_t* rel_flag_out = nullptr, uint64_t bucket_item = ~uint64_t(0)) {
    BatchArgs a = batch_args(bedges, bnegs, P, loss_out, pool);
    if (bk.keys && bucket_item != ~uint64_t(0)) {  // this batch's run of the bucket sort
      a.presorted = 1;
      a.key_mask = bk.mask;
      a.rel_bits = bk.rel_bits;  // the payloads were written with the full batch's layout
      a.skeys = const_cast<uint32_t*>(bk.keys) + bucket_item;
      a.svals = const_cast<uint32_t*>(bk.vals) + bucket_item;
      if (bucket_segs) {  // K4 v2 reads the bucket's segment list
        a.seg_mode = 1;
        a.seg_keys = bk.keys;
        a.seg_vals = bk.vals;
        a.seg_b0 = bucket_item;
        a.seg_batch = (uint32_t)(bucket_item / (uint64_t(opt.batch_size) * (k() + 2)));
      }
    }
    score_bytes_total += score_bytes(P);
    if (rel_grad_out) {  // lock-step rounds: relation gradient only, applied later
      a.grad_rels = rel_grad_out;
      a.grad_rel_flag = rel_flag_out;
      a.side = nullptr;  // the caller applies relation gradients itself
    }
    if (profiling) {
      const int slot = prof_slot(1);
      BatchEvents ev;
      ev.enabled = true;
      for (int i = 0; i < 5; ++i) ev.ev[i] = prof_ev(slot)[i];
      launch_train_batch(a, stream, &ev);
      // algorithmic bytes per phase: score reads the edge and
      // (2 + k + t) rows per positive; the update's row traffic is added
      // from the unique counts at the end of the call.
      kstats[LGD_KSTAT_SCORE].algorithmic_bytes += score_bytes(P);
    } else {
      launch_train_batch(a, stream, nullptr);
    }
    launches += batch_launches(a.node_key_bits);
    if (a.presorted) launches -= 2 + (a.node_key_bits + 7) / 8;
  }

  // Bucket-level presort: every batch's node contributions keyed once as
  // (batch << pool bits) | pool index and sorted in one radix sort over the
  // bucket (train.cu: presort_keys_kernel).  The stable sort keeps each batch's
  // contributions in K3's order, so batch b's run equals its own sort; one
  // large sort runs near HBM speed where ~50 per-batch sorts of 1.8M items
  // are launch- and lookback-bound.  Off (bk.keys = nullptr) for shared
  // negatives and when the keys would not fit 32 bits.
  void presort_bucket(const Pool& pool, uint64_t m, cudaEvent_t* bev, cudaStream_t st) {
    bk = Presorted{};
    bucket_segs = false;
    if (presort && !chunk() && m) {
      const uint64_t B = opt.batch_size;
      const BatchArgs a = batch_args(shuffled.get(), negs.get(), std::min(B, m), nullptr, &pool);
      const uint64_t nb = (m + B - 1) / B;
      const int bbits = bits_for(nb - 1);
      // the relation id rides in the payload when it fits the full batch B
      // (then also every smaller last batch); otherwise no batch carries it
      if (a.node_key_bits + bbits <= 32) {
        const uint64_t items = m * (k() + 2);
        for (int i = 0; i < 2; ++i) {
          bk_keys[i].reserve(items);
          bk_vals[i].reserve(items);
        }
        const size_t tb = bucket_sort_temp_bytes(items);
        if (bk_temp.bytes() < tb) bk_temp.reserve(tb);
        launch_bucket_keys(a, m, B, bk_keys[0].get(), bk_vals[0].get(), st);
        uint32_t* kk[2] = {bk_keys[0].get(), bk_keys[1].get()};
        uint32_t* vv[2] = {bk_vals[0].get(), bk_vals[1].get()};
        const int sel = sort_bucket(bk_temp.get(), bk_temp.bytes(), kk, vv, items,
                                    a.node_key_bits + bbits, st);
        bk.keys = kk[sel];
        bk.vals = vv[sel];
        bk.mask = a.node_key_bits >= 32 ? 0xffffffffu : (1u << a.node_key_bits) - 1u;
        bk.rel_bits = a.rel_bits;
        bk.items = items;
        launches += 1 + 2 + (a.node_key_bits + bbits + 7) / 8;
        if (seg_rows) {  // K4 v2: every batch's segments, listed once for the bucket
          ensure_segments(items, nb);
          launch_long_list(bk.keys, items, uint64_t(B) * (k() + 2), (uint32_t)nb, seg_lists(), st);
          bucket_segs = true;
          launches += 2;
        }
      }
    }
    if (bev) LGD_CUDA(cudaEventRecord(bev[3], st));
  }

  // algorithmic bytes of the score phase: the edge record and
  // (2 + t) rows per positive, plus k rows per positive or per shared chunk
  double score_bytes(uint64_t P) const {
    return double(P) * (12.0 + 4.0 * dim * (2 + (typed() ? 1 : 0))) +
           4.0 * dim * double(batch_negs(P));
  }

  Pool pool_of_state(size_t s) const {
    Pool pool{};
    uint32_t ids[3];
    int np = 0;
    for (uint32_t p : plan.seq.states[s])
      if (p != kNoPartition) ids[np++] = p;
    std::sort(ids, ids + np);
    uint64_t acc = 0;
    for (int i = 0; i < np; ++i) {
      pool.first[i] = part_begin(ids[i]);
      acc += part_rows(ids[i]);
      pool.end_index[i] = acc;
    }
    pool.n = np;
    return pool;
  }

  void check_ready() const {
    if (!E) throw std::invalid_argument("no graph loaded");
    if (!partitioned) throw std::invalid_argument("no partition plan");
    if (!planned) throw std::invalid_argument("no iteration plan");
    if (!tables_ready) throw std::invalid_argument("embedding store not initialised");
    if (typed() && R == 0)
      throw std::invalid_argument("typed model on a store without relation embeddings");
    if (opt.batch_size == 0) throw std::invalid_argument("batch size must be positive");
    if (opt.negatives == 0)
      throw std::invalid_argument("at least one negative per positive required");
    check_shared();
  }

  // One bucket of work: bucket (bi, bj), its RNG stream index g (the
  // position in the schedule, pipeline.cpp:296) and its negative pool.
  struct WorkItem {
    uint32_t bi, bj;
    uint64_t g;
    Pool pool;
  };

  Pool pool_of_parts(const uint32_t* parts, int count) const {
    uint32_t ids[3];
    int np = 0;
    for (int i = 0; i < count; ++i)
      if (parts[i] != kNoPartition) {
        if (parts[i] >= n) throw std::invalid_argument("pool partition out of range");
        ids[np++] = parts[i];
      }
    if (np == 0) throw std::invalid_argument("empty negative pool");
    std::sort(ids, ids + np);
    Pool pool{};
    uint64_t acc = 0;
    for (int i = 0; i < np; ++i) {
      pool.first[i] = part_begin(ids[i]);
      acc += part_rows(ids[i]);
      pool.end_index[i] = acc;
    }
    pool.n = np;
    return pool;
  }

  std::vector<WorkItem> plan_items(uint64_t g_begin, uint64_t g_end) const {
    std::vector<WorkItem> items;
    const uint64_t G = plan.bucket_order.size();
    g_end = std::min(g_end, G);
    size_t st = 0;
    for (uint64_t g = g_begin; g < g_end; ++g) {
      while (st + 1 < plan.seq.states.size() && g >= plan.state_offsets[st + 1]) ++st;
      const auto [bi, bj] = plan.bucket_order[g];
      items.push_back({bi, bj, g, pool_of_state(st)});
    }
    return items;
  }

  uint64_t bucket_size(const WorkItem& it, uint64_t* off = nullptr) const {
    const uint64_t b = uint64_t(it.bi) * n + it.bj;
    if (off) *off = offsets[b];
    return offsets[b + 1] - offsets[b];
  }

  // Shuffle draws + permutation + gather, then the bucket's m*k negative
  // draws, all from the bucket's stream (pipeline.cpp:296-308).
  void prepare_bucket(const WorkItem& it, uint32_t epoch, const uint32_t* bucket_edges, uint64_t m,
                      cudaEvent_t* bev, cudaStream_t st) {
    StreamSlot slot{xo_seed(derive_seed(opt.seed, kTagBucket, epoch, it.g)), pos.get(),
                    reject.get()};
    if (bev) LGD_CUDA(cudaEventRecord(bev[0], st));
    LGD_CUDA(cudaMemsetAsync(pos.get(), 0, sizeof(uint64_t), st));
    if (opt.shuffle) {
      launch_shuffle_draws(slot, m, H.get(), st);
      ShuffleScratch s{sh_keys_in.get(), sh_vals_in.get(), sh_keys_out.get(), sh_vals_out.get(),
                       sh_ptr.get(),     sh_G.get(),       sh_temp.get(),     sh_temp.bytes()};
      launch_shuffle_permutation(H.get(), m, s, perm.get(), st);
      launch_gather_edges(bucket_edges, perm.get(), m, shuffled.get(), st);
      launches += 2 + 5 + 2 + (bits_for(m) + 7) / 8 + 1;
    } else {
      launch_gather_edges(bucket_edges, nullptr, m, shuffled.get(), st);
      launches += 1;
    }
  }
  void sample_bucket(const WorkItem& it, uint32_t epoch, uint64_t m, cudaEvent_t* bev,
                     cudaStream_t st) {
    (void)epoch;
    StreamSlot slot{xo_seed(derive_seed(opt.seed, kTagBucket, epoch, it.g)), pos.get(),
                    reject.get()};
    if (bev) LGD_CUDA(cudaEventRecord(bev[1], st));
    launch_sample_nodes(slot, bucket_negs(m), it.pool, negs.get(), st);
    launches += 2;
    if (bev) LGD_CUDA(cudaEventRecord(bev[2], st));
  }

  // the largest bucket of the partition plan: scratch is sized for it once,
  // so no buffer grows (cudaFree + cudaMalloc, a device sync) mid-epoch
  uint64_t max_bucket() const {
    uint64_t mx = 0;
    for (size_t b = 0; b + 1 < offsets.size(); ++b) mx = std::max(mx, offsets[b + 1] - offsets[b]);
    return mx;
  }

  void reserve_for(const std::vector<WorkItem>& items, uint64_t* total_batches) {
    uint64_t max_m = max_bucket(), tb = 0;
    for (const auto& it : items) {
      const uint64_t m = bucket_size(it);
      tb += (m + opt.batch_size - 1) / opt.batch_size;
    }
    ensure_bucket(max_m);
    ensure_batch(std::min<uint64_t>(opt.batch_size, std::max<uint64_t>(max_m, 1)));
    if (presort && !chunk() && max_m) {  // bucket sort buffers, sized once
      const uint64_t items = max_m * (k() + 2);
      for (int i = 0; i < 2; ++i) {
        bk_keys[i].reserve(items);
        bk_vals[i].reserve(items);
      }
      bk_temp.reserve(bucket_sort_temp_bytes(items));
      if (seg_rows) ensure_segments(items, (max_m + opt.batch_size - 1) / opt.batch_size);
    }
    batch_losses.reserve(std::max<uint64_t>(tb, 1));
    if (total_batches) *total_batches = tb;
  }

  void fill_result(lgd_epoch_result* out, uint64_t nb, uint64_t edges_trained, uint64_t buckets,
                   uint64_t h2d_bytes, std::chrono::steady_clock::time_point t0) {
    LGD_CUDA(cudaEventRecord(ev_end, stream));
    LGD_CUDA(cudaStreamSynchronize(stream));
    prof_flush();
    std::vector<double> losses(nb);
    if (nb)
      LGD_CUDA(cudaMemcpy(losses.data(), batch_losses.get(), nb * 8, cudaMemcpyDeviceToHost));
    unsigned long long cnt[2] = {0, 0};
    LGD_CUDA(cudaMemcpy(cnt, counters.get(), sizeof cnt, cudaMemcpyDeviceToHost));
    double loss_sum = 0.0;
    for (double l : losses) loss_sum += l;  // pipeline.cpp:309, batch order
    float dev_ms = 0;
    LGD_CUDA(cudaEventElapsedTime(&dev_ms, ev_begin, ev_end));
    if (profiling) {
      kstats[LGD_KSTAT_UPDATE].algorithmic_bytes += 16.0 * dim * double(cnt[0]);
      kstats[LGD_KSTAT_REL].algorithmic_bytes += 16.0 * dim * double(cnt[1]);
    }
    if (out) {
      const uint32_t kk = k();
      std::memset(out, 0, sizeof *out);
      out->loss_sum = loss_sum;
      out->edges_trained = edges_trained;
      out->buckets_trained = buckets;
      out->loss_per_edge = edges_trained ? loss_sum / double(edges_trained) : 0.0;
      out->batches = nb;
      out->wall_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      out->device_ms = dev_ms;
      out->unique_nodes = cnt[0];
      out->unique_rels = cnt[1];
      out->h2d_bytes = h2d_bytes;
      out->d2h_bytes = nb * 8 + sizeof cnt;
      (void)kk;
      out->algorithmic_bytes = score_bytes_total + 16.0 * dim * double(cnt[0] + cnt[1]);
    }
  }

  // Trains a list of buckets in order.  host_bucketed: optional host copy
  // (pinned for full speed) of the edges in bucket order; each bucket is then
  // streamed H2D on a side stream, one bucket ahead of the compute.
  // batch_limit: at most that many batches per bucket (a bounded prefix of the
  // reference loop, for parity at full scale); node_trace (device, one slot
  // per batch): the running unique-node counter after every batch.
  // hook(i, before): called as bucket i of `items` is queued (before its
  // first kernel) and after its last batch is queued, empty buckets
  // included (the round runner orders partition hand-offs there).
  // finish = false: return with the work queued; finish_items() collects.
  struct Pending {
    uint64_t nb = 0, edges = 0, buckets = 0, h2d = 0;
    std::chrono::steady_clock::time_point t0;
  } pending;
  void train_items(uint32_t epoch, const std::vector<WorkItem>& items, lgd_epoch_result* out,
                   const uint32_t* host_bucketed = nullptr, uint64_t batch_limit = ~uint64_t(0),
                   unsigned long long* node_trace = nullptr,
                   const std::function<void(size_t, bool)>* hook = nullptr, bool finish = true) {
    check_ready();
    const auto t0 = std::chrono::steady_clock::now();
    reserve_for(items, nullptr);
    const uint64_t max_m = max_bucket();
    auto next_nonempty = [&](size_t i) {
      while (i < items.size() && bucket_size(items[i]) == 0) ++i;
      return i;
    };
    int stage = 0;
    uint64_t h2d_bytes = 0;
    auto issue_copy = [&](size_t i, int slot) {
      uint64_t off;
      const uint64_t m = bucket_size(items[i], &off);
      LGD_CUDA(cudaStreamWaitEvent(copy_stream, stage_free[slot], 0));
      LGD_CUDA(cudaMemcpyAsync(staging[slot].get(), host_bucketed + 3 * off, m * 12,
                               cudaMemcpyHostToDevice, copy_stream));
      LGD_CUDA(cudaEventRecord(copy_done[slot], copy_stream));
      h2d_bytes += m * 12;
    };
    LGD_CUDA(cudaMemsetAsync(counters.get(), 0, 2 * sizeof(unsigned long long), stream));
    LGD_CUDA(cudaEventRecord(ev_begin, stream));
    score_bytes_total = 0.0;
    if (host_bucketed) {
      staging[0].reserve(max_m * 3);
      staging[1].reserve(max_m * 3);
      const size_t i0 = next_nonempty(0);
      LGD_CUDA(cudaEventRecord(stage_free[0], stream));
      LGD_CUDA(cudaEventRecord(stage_free[1], stream));
      if (i0 < items.size()) issue_copy(i0, 0);
    }
    uint64_t nb = 0, edges_trained = 0, buckets = 0;
    // bucket i's shuffle / sample / presort into the members' buffer set,
    // on `ps`: prep_stream (overlapped with the previous bucket's batches)
    // or the training stream itself
    const bool ovl = overlap_prep && prep_stream;
    cudaStream_t ps = ovl ? prep_stream : stream;
    if (ovl) {
      reserve_alt();
      // neither set is rewritten before the stream's earlier readers finish
      LGD_CUDA(cudaEventRecord(ev_consumed[0], stream));
      LGD_CUDA(cudaEventRecord(ev_consumed[1], stream));
    }
    auto prep = [&](size_t i) {
      const WorkItem& it = items[i];
      uint64_t off;
      const uint64_t m = bucket_size(it, &off);
      cudaEvent_t* bev = profiling ? prof_ev(prof_slot(2)) : nullptr;
      const uint32_t* bucket_edges = edges_bucketed.get() + 3 * off;
      if (ovl) LGD_CUDA(cudaStreamWaitEvent(ps, ev_consumed[set_id], 0));
      if (host_bucketed) {
        LGD_CUDA(cudaStreamWaitEvent(ps, copy_done[stage], 0));
        bucket_edges = staging[stage].get();
        const size_t in = next_nonempty(i + 1);
        if (in < items.size()) issue_copy(in, stage ^ 1);
      }
      prepare_bucket(it, epoch, bucket_edges, m, bev, ps);
      if (host_bucketed) {
        LGD_CUDA(cudaEventRecord(stage_free[stage], ps));
        stage ^= 1;
      }
      sample_bucket(it, epoch, m, bev, ps);
      presort_bucket(it.pool, m, bev, ps);
      if (ovl) LGD_CUDA(cudaEventRecord(ev_prepped[set_id], ps));
    };
    if (ovl && next_nonempty(0) < items.size()) prep(next_nonempty(0));
    for (size_t idx = 0; idx < items.size(); ++idx) {
      const WorkItem& it = items[idx];
      const uint64_t m = bucket_size(it);
      if (hook) (*hook)(idx, true);
      if (m == 0) {  // pipeline.cpp:291, before the RNG is created
        if (hook) (*hook)(idx, false);
        continue;
      }
      if (ovl)
        LGD_CUDA(cudaStreamWaitEvent(stream, ev_prepped[set_id], 0));
      else
        prep(idx);
      uint64_t done = 0;
      for (uint64_t o = 0, b = 0; o < m && b < batch_limit; o += opt.batch_size, ++b) {
        const uint64_t P = std::min<uint64_t>(opt.batch_size, m - o);
        run_batch(shuffled.get() + 3 * o, negs.get() + (o / opt.batch_size) * batch_negs(opt.batch_size),
                  P, batch_losses.get() + nb, &it.pool, nullptr, nullptr, o * (k() + 2));
        if (node_trace)
          LGD_CUDA(cudaMemcpyAsync(node_trace + nb, counters.get(), sizeof(unsigned long long),
                                   cudaMemcpyDeviceToDevice, stream));
        ++nb;
        done += P;
      }
      if (ovl) {  // the next bucket's prep overlaps these batches
        LGD_CUDA(cudaEventRecord(ev_consumed[set_id], stream));
        const size_t in = next_nonempty(idx + 1);
        if (in < items.size()) {
          swap_sets();
          prep(in);
        }
      }
      edges_trained += done;
      ++buckets;
      if (hook) (*hook)(idx, false);
    }
    pending = Pending{nb, edges_trained, buckets, h2d_bytes, t0};
    if (finish) finish_items(out);
  }
  void finish_items(lgd_epoch_result* out) {
    fill_result(out, pending.nb, pending.edges, pending.buckets, pending.h2d, pending.t0);
  }

  void train_range(uint32_t epoch, uint64_t g_begin, uint64_t g_end, lgd_epoch_result* out,
                   const uint32_t* host_bucketed = nullptr) {
    if (!host_bucketed) host_bucketed = host_edges;
    check_ready();
    train_items(epoch, plan_items(g_begin, g_end), out, host_bucketed);
  }

  // ---- lock-step rounds (multi-GPU, typed models): this rank's batches are
  // run one at a time; after each, the caller sums the dense relation
  // gradient [R x (d+1)] (last column: touched flag) across ranks and hands
  // the sum back for one identical relation Adagrad step on every rank.
  std::vector<WorkItem> round_items;
  std::vector<uint64_t> round_first_batch;  // per item, prefix of batch counts
  uint64_t round_batches = 0, round_nb = 0, round_edges = 0, round_buckets = 0;
  uint32_t round_epoch = 0;
  size_t round_prepared = ~size_t(0);
  // lgd_set_stream_ordered: round_step / round_apply_relations return without
  // draining the stream; the caller orders its collective on it instead
  bool stream_ordered = false;
  std::chrono::steady_clock::time_point round_t0;
  DevBuf<double> rel_grad;
  DevBuf<uint8_t> rel_flag;

  uint64_t round_begin(uint32_t epoch, std::vector<WorkItem> items) {
    check_ready();
    round_t0 = std::chrono::steady_clock::now();
    round_items = std::move(items);
    round_first_batch.assign(round_items.size() + 1, 0);
    for (size_t i = 0; i < round_items.size(); ++i) {
      const uint64_t m = bucket_size(round_items[i]);
      round_first_batch[i + 1] = round_first_batch[i] + (m + opt.batch_size - 1) / opt.batch_size;
    }
    round_batches = round_first_batch.back();
    reserve_for(round_items, nullptr);
    rel_grad.reserve(std::max<uint64_t>(R, 1) * dim);
    rel_flag.reserve(std::max<uint64_t>(R, 1));
    round_epoch = epoch;
    round_prepared = ~size_t(0);
    round_nb = round_edges = round_buckets = 0;
    round_h2d = 0;
    score_bytes_total = 0.0;
    LGD_CUDA(cudaMemsetAsync(counters.get(), 0, 2 * sizeof(unsigned long long), stream));
    LGD_CUDA(cudaEventRecord(ev_begin, stream));
    return round_batches;
  }

  // Lock-step batch `step` of this rank (a no-op past its last batch); the
  // dense relation gradient lands in rel_out [R x (d+1)] (device).
  void round_step(uint64_t step, double* rel_out) {
    const uint64_t rows = std::max<uint64_t>(R, 1);
    LGD_CUDA(cudaMemsetAsync(rel_grad.get(), 0, rows * dim * 8, stream));
    LGD_CUDA(cudaMemsetAsync(rel_flag.get(), 0, rows, stream));
    if (step < round_batches) {
      const size_t i = std::upper_bound(round_first_batch.begin(), round_first_batch.end(), step) -
                       round_first_batch.begin() - 1;
      const WorkItem& it = round_items[i];
      uint64_t off;
      const uint64_t m = bucket_size(it, &off);
      if (round_prepared != i) {
        const uint32_t* src = edges_bucketed.get() + 3 * off;
        if (host_edges) {  // this step's bucket from host memory
          staging[0].reserve(max_bucket() * 3);
          LGD_CUDA(cudaMemcpyAsync(staging[0].get(), host_edges + 3 * off, m * 12,
                                   cudaMemcpyHostToDevice, stream));
          src = staging[0].get();
          round_h2d += m * 12;
        }
        prepare_bucket(it, round_epoch, src, m, nullptr, stream);
        sample_bucket(it, round_epoch, m, nullptr, stream);
        presort_bucket(it.pool, m, nullptr, stream);
        round_prepared = i;
        round_edges += m;
        ++round_buckets;
      }
      const uint64_t o = (step - round_first_batch[i]) * opt.batch_size;
      const uint64_t P = std::min<uint64_t>(opt.batch_size, m - o);
      run_batch(shuffled.get() + 3 * o, negs.get() + (o / opt.batch_size) * batch_negs(opt.batch_size),
                P, batch_losses.get() + round_nb,
                &it.pool, typed() ? rel_grad.get() : nullptr, typed() ? rel_flag.get() : nullptr,
                o * (k() + 2));
      ++round_nb;
    }
    if (rel_out) launch_rel_pack(rel_grad.get(), rel_flag.get(), R, dim, rel_out, stream);
    if (!stream_ordered) LGD_CUDA(cudaStreamSynchronize(stream));
  }

  void round_apply_relations(const double* summed) {
    if (typed() && R) {
      launch_rel_apply(summed, rel_theta.get(), rel_state.get(), R, dim, opt.learning_rate,
                       opt.adagrad_epsilon, stream);
      if (!stream_ordered) LGD_CUDA(cudaStreamSynchronize(stream));
    }
  }

  void round_end(lgd_epoch_result* out) {
    fill_result(out, round_nb, round_edges, round_buckets, round_h2d, round_t0);
  }

  // Operator-level batch on host inputs (validated like batch_loss,
  // train.cpp:217-241).
  void upload_batch(const uint32_t* h_edges, uint64_t P, const uint32_t* h_negs) {
    if (!tables_ready) throw std::invalid_argument("embedding store not initialised");
    if (opt.negatives == 0)
      throw std::invalid_argument("at least one negative per positive required");
    check_shared();
    const uint64_t nn = batch_negs(P);
    for (uint64_t q = 0; q < nn; ++q)
      if (h_negs[q] >= V)
        throw std::out_of_range("node " + std::to_string(h_negs[q]) + " is not resident");
    for (uint64_t p = 0; p < P; ++p) {
      const uint32_t s = h_edges[3 * p], r = h_edges[3 * p + 1], t = h_edges[3 * p + 2];
      if (s >= V || t >= V) throw std::out_of_range("node " + std::to_string(s >= V ? s : t) +
                                                    " is not resident");
      if (typed()) {
        if (r == LGD_NO_RELATION)
          throw std::invalid_argument("typed model requires a relation id on every edge");
        if (r >= R) throw std::out_of_range("relation id out of range");
      }
    }
    op_edges.reserve(std::max<uint64_t>(P * 3, 3));
    op_negs.reserve(std::max<uint64_t>(nn, 1));
    if (P) {
      LGD_CUDA(cudaMemcpyAsync(op_edges.get(), h_edges, P * 12, cudaMemcpyHostToDevice, stream));
      LGD_CUDA(cudaMemcpyAsync(op_negs.get(), h_negs, nn * 4, cudaMemcpyHostToDevice, stream));
    }
    ensure_batch(std::max<uint64_t>(P, 1));
    batch_losses.reserve(1);
  }
};

