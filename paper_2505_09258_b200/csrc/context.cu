// context.cu -- the C ABI (include/legend_b200.h) and the host epoch driver.
//
// The driver is the real-train branch of run_epoch (pipeline.cpp:273-322)
// with every partition resident in HBM: the SSD tier, NVMe simulation and
// state-boundary swaps of the reference become a change of the sampling
// pool (the partitions of the current plan state), exactly the reference's
// own in-memory restatement (test_pipeline.cpp:227-269).  Per non-empty
// bucket g of bucket_order:
//   stream  Rng(derive_seed(seed, "bukt", epoch, g))       pipeline.cpp:296
//   K2      m-1 Fisher-Yates draws, then m*k negative draws (one stream,
//           consumed in the reference's order; device offset counter)
//   K1      permutation from the draws + gather of the bucket's edges
//   per batch of P edges: K3 score -> sort -> K4 update -> relations
// Nothing is synchronised with the host inside an epoch.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>
#include <cstdlib>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

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
thread_local std::string g_last_error;
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace lgd

namespace {

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    LGD_CUDA(cudaGetDevice(&prev));
    if (prev != dev) LGD_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

constexpr int kProfRing = 256;

}  // namespace

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
  DevBuf<float> sn_A, sn_AT, sn_B, sn_BT, sn_rowmax, sn_rowinv, sn_G;
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
  DevBuf<uint32_t> seg_start, batch_seg, seg_nseg;
  DevBuf<unsigned int> seg_work;
  DevBuf<unsigned char> seg_temp;
  bool bucket_segs = false;  // the current bucket's segment list is built
  struct Presorted {
    const uint32_t* keys = nullptr;
    const uint32_t* vals = nullptr;
    uint32_t mask = 0;
    int rel_bits = 0;  // payload layout of the whole bucket
    uint64_t items = 0;
  } bk;
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
  double eval_ms = 0.0;  // device time of the last lgd_evaluate (profiling mode)
  size_t l2_persist = 0, l2_window_max = 0;  // L2 set-aside for the snapshot rows
  // optional host copy of the bucket-ordered edges (lgd_set_host_edges): the
  // bucket lists and rounds then stream every bucket H2D instead of reading
  // the device copy
  const uint32_t* host_edges = nullptr;
  uint64_t round_h2d = 0;
  double score_bytes_total = 0.0;  // algorithmic score-phase bytes since the call began

  ~lgd_context() {
    cudaSetDevice(device);
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
    for (auto e : {copy_done[0], copy_done[1], stage_free[0], stage_free[1]})
      if (e) cudaEventDestroy(e);
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
      sn_B.reserve(sh.nch * sh.kpad * sh.dpad);
      sn_BT.reserve(sh.nch * sh.kpad * sh.dpad);
      sn_rowmax.reserve(rows);
      sn_rowinv.reserve(rows);
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
    part_first.reserve(chunks * dim);
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
    seg_start.reserve(items + 1);
    batch_seg.reserve(nb + 1);
    seg_work.reserve(std::max<uint64_t>(nb, 1));
    seg_nseg.reserve(1);
    const size_t tb = segment_list_temp_bytes(items);
    if (seg_temp.bytes() < tb) seg_temp.reserve(tb);
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
    a.edges = bedges;
    a.negs = bnegs;
    a.theta = theta.get();
    a.state = state.get();
    a.rel_theta = rel_theta.get();
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
    a.seg_mode = seg_rows ? 2 : 0;  // run_batch switches to the bucket's list
    a.seg_start = seg_start.get();
    a.batch_seg = batch_seg.get();
    a.seg_work = seg_work.get();
    a.seg_nseg = seg_nseg.get();
    a.seg_temp = seg_temp.get();
    a.seg_temp_bytes = seg_temp.bytes();
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
      a.sh_rowmax = sn_rowmax.get();
      a.sh_rowinv = sn_rowinv.get();
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
        a.seg_n = bk.items;
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
  void presort_bucket(const Pool& pool, uint64_t m, cudaEvent_t* bev) {
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
        launch_bucket_keys(a, m, B, bk_keys[0].get(), bk_vals[0].get(), stream);
        uint32_t* kk[2] = {bk_keys[0].get(), bk_keys[1].get()};
        uint32_t* vv[2] = {bk_vals[0].get(), bk_vals[1].get()};
        const int sel = sort_bucket(bk_temp.get(), bk_temp.bytes(), kk, vv, items,
                                    a.node_key_bits + bbits, stream);
        bk.keys = kk[sel];
        bk.vals = vv[sel];
        bk.mask = a.node_key_bits >= 32 ? 0xffffffffu : (1u << a.node_key_bits) - 1u;
        bk.rel_bits = a.rel_bits;
        bk.items = items;
        launches += 1 + 2 + (a.node_key_bits + bbits + 7) / 8;
        if (seg_rows) {  // K4 v2: every batch's segments, listed once for the bucket
          ensure_segments(items, nb);
          LGD_CUDA(cudaMemsetAsync(seg_work.get(), 0, nb * sizeof(unsigned int), stream));
          launch_segment_list(bk.keys, items, a.node_key_bits, (uint32_t)nb, seg_start.get(),
                              batch_seg.get(), seg_nseg.get(), seg_temp.get(), seg_temp.bytes(),
                              sm_count, stream);
          bucket_segs = true;
          launches += 3;
        }
      }
    }
    if (bev) LGD_CUDA(cudaEventRecord(bev[3], stream));
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
                      cudaEvent_t* bev) {
    StreamSlot slot{xo_seed(derive_seed(opt.seed, kTagBucket, epoch, it.g)), pos.get(),
                    reject.get()};
    if (bev) LGD_CUDA(cudaEventRecord(bev[0], stream));
    LGD_CUDA(cudaMemsetAsync(pos.get(), 0, sizeof(uint64_t), stream));
    if (opt.shuffle) {
      launch_shuffle_draws(slot, m, H.get(), stream);
      ShuffleScratch s{sh_keys_in.get(), sh_vals_in.get(), sh_keys_out.get(), sh_vals_out.get(),
                       sh_ptr.get(),     sh_G.get(),       sh_temp.get(),     sh_temp.bytes()};
      launch_shuffle_permutation(H.get(), m, s, perm.get(), stream);
      launch_gather_edges(bucket_edges, perm.get(), m, shuffled.get(), stream);
      launches += 2 + 5 + 2 + (bits_for(m) + 7) / 8 + 1;
    } else {
      launch_gather_edges(bucket_edges, nullptr, m, shuffled.get(), stream);
      launches += 1;
    }
  }
  void sample_bucket(const WorkItem& it, uint32_t epoch, uint64_t m, cudaEvent_t* bev) {
    (void)epoch;
    StreamSlot slot{xo_seed(derive_seed(opt.seed, kTagBucket, epoch, it.g)), pos.get(),
                    reject.get()};
    if (bev) LGD_CUDA(cudaEventRecord(bev[1], stream));
    launch_sample_nodes(slot, bucket_negs(m), it.pool, negs.get(), stream);
    launches += 2;
    if (bev) LGD_CUDA(cudaEventRecord(bev[2], stream));
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
  void train_items(uint32_t epoch, const std::vector<WorkItem>& items, lgd_epoch_result* out,
                   const uint32_t* host_bucketed = nullptr, uint64_t batch_limit = ~uint64_t(0),
                   unsigned long long* node_trace = nullptr) {
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
    const uint32_t kk = k();
    for (size_t idx = 0; idx < items.size(); ++idx) {
      const WorkItem& it = items[idx];
      uint64_t off;
      const uint64_t m = bucket_size(it, &off);
      if (m == 0) continue;  // pipeline.cpp:291, before the RNG is created
      cudaEvent_t* bev = profiling ? prof_ev(prof_slot(2)) : nullptr;
      const uint32_t* bucket_edges = edges_bucketed.get() + 3 * off;
      if (host_bucketed) {
        LGD_CUDA(cudaStreamWaitEvent(stream, copy_done[stage], 0));
        bucket_edges = staging[stage].get();
        const size_t in = next_nonempty(idx + 1);
        if (in < items.size()) issue_copy(in, stage ^ 1);
      }
      prepare_bucket(it, epoch, bucket_edges, m, bev);
      if (host_bucketed) {
        LGD_CUDA(cudaEventRecord(stage_free[stage], stream));
        stage ^= 1;
      }
      sample_bucket(it, epoch, m, bev);
      presort_bucket(it.pool, m, bev);
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
      edges_trained += done;
      ++buckets;
    }
    fill_result(out, nb, edges_trained, buckets, h2d_bytes, t0);
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
        prepare_bucket(it, round_epoch, src, m, nullptr);
        sample_bucket(it, round_epoch, m, nullptr);
        presort_bucket(it.pool, m, nullptr);
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

// ============================================================== C ABI ====
extern "C" {

const char* lgd_last_error(void) { return g_last_error.c_str(); }

int lgd_create(lgd_context** out, int model_kind, uint32_t dim, const lgd_train_options* options,
               int device) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null output pointer");
    *out = nullptr;
    if (model_kind < 0 || model_kind > 3) throw std::invalid_argument("unknown score model");
    if (dim == 0) throw std::invalid_argument("embedding dimension must be positive");
    if (model_kind == LGD_MODEL_COMPLEX && dim % 2 != 0)
      throw std::invalid_argument("complex model requires an even dimension");
    if ((model_kind == LGD_MODEL_COMPLEX ? dim / 2 : dim) > 256)
      throw std::invalid_argument("embedding dimension too large (max 256, ComplEx 512)");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw lgd::cuda_error("no CUDA device: the B200 path has no CPU fallback");
    if (device < 0 || device >= count) throw std::invalid_argument("bad device ordinal");
    DeviceGuard g(device);
    auto* c = new lgd_context();
    try {
      c->device = device;
      c->kind = model_kind;
      c->dim = dim;
      if (options) {
        c->opt = *options;
      } else {
        c->opt = lgd_train_options{0.1, 1e-10, 100000, 16, 1, 0, 0};
      }
      LGD_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
      LGD_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      {  // L2 set-aside for the snapshot rows (LGD_L2_PERSIST=0 disables)
        int pmax = 0, wmax = 0;
        cudaDeviceGetAttribute(&pmax, cudaDevAttrMaxPersistingL2CacheSize, device);
        cudaDeviceGetAttribute(&wmax, cudaDevAttrMaxAccessPolicyWindowSize, device);
        const char* env = std::getenv("LGD_L2_PERSIST");
        // 48 MB for the f32 snapshot rows; none when K4 reads the 2x wider f64
        // IR1 rows (k4_ir1: FM +1.1%, Friendster +1.3% without the window)
        const size_t want_mb = env ? std::strtoull(env, nullptr, 10) : (k4_ir1(model_kind) ? 0 : 48);
        if (want_mb && pmax > 0 && wmax > 0) {
          const size_t want = std::min<size_t>((size_t)pmax, want_mb << 20);
          if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
            c->l2_persist = want;
            c->l2_window_max = (size_t)wmax;
          }
        }
        cudaGetLastError();  // the set-aside is an optimisation only
      }
      if (const char* env = std::getenv("LGD_PRESORT")) c->presort = std::strtol(env, nullptr, 10) != 0;
      if (const char* env = std::getenv("LGD_K4")) c->seg_rows = std::strtol(env, nullptr, 10) != 1;
      if (const char* env = std::getenv("LGD_K4_IR1")) c->ir1_rows = std::strtol(env, nullptr, 10) != 0;
      LGD_CUDA(cudaEventCreate(&c->ev_begin));
      LGD_CUDA(cudaEventCreate(&c->ev_end));
      LGD_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
      {  // the relation pass / loss reduction is small and overlaps K4, which
         // fills every SM: at the highest priority its blocks are scheduled as
         // soon as K4 blocks retire instead of after K4's whole grid
        int lo = 0, hi = 0;
        LGD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        LGD_CUDA(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, hi));
      }
      LGD_CUDA(cudaEventCreateWithFlags(&c->ev_scored, cudaEventDisableTiming));
      LGD_CUDA(cudaEventCreateWithFlags(&c->ev_rel, cudaEventDisableTiming));
      for (auto* e : {&c->copy_done[0], &c->copy_done[1], &c->stage_free[0], &c->stage_free[1]})
        LGD_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      c->pos.reserve(1);
      c->reject.reserve(1);
      LGD_CUDA(cudaMemset(c->reject.get(), 0xff, sizeof(unsigned long long)));
      c->counters.reserve(2);
      jump_tables(device);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

void lgd_destroy(lgd_context* ctx) { delete ctx; }

int lgd_set_options(lgd_context* ctx, const lgd_train_options* options) {
  return guarded([&] {
    if (!ctx || !options) throw std::invalid_argument("null argument");
    ctx->opt = *options;
  });
}

int lgd_set_graph(lgd_context* ctx, const uint32_t* edges, uint64_t num_edges, uint64_t num_nodes,
                  uint64_t num_relations) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (num_nodes == 0 || num_nodes > 0xffffffffull)
      throw std::invalid_argument("node count must be in [1, 2^32)");
    if (num_edges >= 0xffffffffull) throw std::invalid_argument("too many edges (max 2^32-1)");
    for (uint64_t e = 0; e < num_edges; ++e) {
      if (edges[3 * e] >= num_nodes || edges[3 * e + 2] >= num_nodes)
        throw std::invalid_argument("edge endpoint outside the node range");
      const uint32_t r = edges[3 * e + 1];
      if (num_relations && r >= num_relations)
        throw std::invalid_argument("edge relation outside the relation range");
    }
    DeviceGuard g(ctx->device);
    ctx->edges.reserve(std::max<uint64_t>(num_edges * 3, 3));
    if (num_edges)
      LGD_CUDA(cudaMemcpyAsync(ctx->edges.get(), edges, num_edges * 12, cudaMemcpyHostToDevice,
                               ctx->stream));
    ctx->V = num_nodes;
    ctx->R = num_relations;
    ctx->E = num_edges;
    ctx->partitioned = false;
    ctx->tables_ready = false;
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int lgd_generate_graph(lgd_context* ctx, uint64_t num_nodes, uint64_t num_relations,
                       uint64_t num_edges, double zipf_exponent, uint64_t seed) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (num_nodes == 0 || num_nodes > 0xffffffffull)
      throw std::invalid_argument("node count must be in [1, 2^32)");
    if (num_edges >= 0xffffffffull) throw std::invalid_argument("too many edges (max 2^32-1)");
    DeviceGuard g(ctx->device);
    ctx->edges.reserve(std::max<uint64_t>(num_edges * 3, 3));
    launch_generate_powerlaw(num_nodes, num_relations, num_edges, zipf_exponent, seed,
                             ctx->edges.get(), ctx->stream);
    ctx->V = num_nodes;
    ctx->R = num_relations;
    ctx->E = num_edges;
    ctx->partitioned = false;
    ctx->tables_ready = false;
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int lgd_get_graph(lgd_context* ctx, uint32_t* edges_out) {
  return guarded([&] {
    if (!ctx || !edges_out) throw std::invalid_argument("null argument");
    DeviceGuard g(ctx->device);
    if (ctx->E)
      LGD_CUDA(cudaMemcpy(edges_out, ctx->edges.get(), ctx->E * 12, cudaMemcpyDeviceToHost));
  });
}

int lgd_make_partition_plan(lgd_context* ctx, uint32_t n, uint64_t* bucket_offsets_out,
                            uint64_t* edge_order_out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    // graph.cpp:121-123
    if (n < 1) throw std::invalid_argument("partition count must be >= 1");
    if (n > ctx->V) throw std::invalid_argument("partition count exceeds node count");
    if (ctx->E == 0) throw std::invalid_argument("graph has no edges");
    DeviceGuard g(ctx->device);
    const uint64_t E = ctx->E, buckets = uint64_t(n) * n;
    const uint64_t stride = (ctx->V + n - 1) / n;
    DevBuf<uint32_t> keys, iota, skeys, order;
    DevBuf<unsigned long long> counts;
    DevBuf<unsigned char> temp;
    keys.reserve(E);
    iota.reserve(E);
    skeys.reserve(E);
    order.reserve(E);
    counts.reserve(buckets);
    LGD_CUDA(cudaMemsetAsync(counts.get(), 0, buckets * 8, ctx->stream));
    launch_bucket_keys(ctx->edges.get(), E, stride, n, keys.get(), iota.get(), counts.get(),
                       ctx->stream);
    const int bits = bits_for(buckets - 1);
    size_t bytes = 0;
    LGD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.get(), skeys.get(), iota.get(),
                                             order.get(), (int64_t)E, 0, bits, ctx->stream));
    temp.reserve(bytes);
    LGD_CUDA(cub::DeviceRadixSort::SortPairs(temp.get(), bytes, keys.get(), skeys.get(),
                                             iota.get(), order.get(), (int64_t)E, 0, bits,
                                             ctx->stream));
    keys.release();
    skeys.release();
    iota.release();
    temp.release();
    ctx->edges_bucketed.reserve(E * 3);
    launch_gather_u32x3(ctx->edges.get(), order.get(), E, ctx->edges_bucketed.get(), ctx->stream);
    std::vector<unsigned long long> h(buckets);
    LGD_CUDA(cudaMemcpyAsync(h.data(), counts.get(), buckets * 8, cudaMemcpyDeviceToHost,
                             ctx->stream));
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->offsets.assign(buckets + 1, 0);
    for (uint64_t b = 0; b < buckets; ++b) ctx->offsets[b + 1] = ctx->offsets[b] + h[b];
    if (bucket_offsets_out)
      std::memcpy(bucket_offsets_out, ctx->offsets.data(), (buckets + 1) * 8);
    if (edge_order_out) {
      std::vector<uint32_t> o(E);
      LGD_CUDA(cudaMemcpy(o.data(), order.get(), E * 4, cudaMemcpyDeviceToHost));
      for (uint64_t i = 0; i < E; ++i) edge_order_out[i] = o[i];
    }
    ctx->n = n;
    ctx->stride = stride;
    ctx->partitioned = true;
    if (n <= 3) {  // one all-resident state (plan_loading_order needs n >= 4)
      ctx->plan = single_state_plan(n);
      ctx->planned = true;
    } else if (!ctx->planned || ctx->plan.seq.n != n) {
      ctx->plan = make_iteration_plan(make_loading_order(n), n);
      ctx->planned = true;
    }
  });
}

int lgd_set_partition_plan(lgd_context* ctx, uint32_t n, const uint64_t* bucket_offsets,
                           const uint64_t* edge_order) {
  return guarded([&] {
    if (!ctx || !bucket_offsets || !edge_order) throw std::invalid_argument("null argument");
    if (n < 1 || n > ctx->V) throw std::invalid_argument("bad partition count");
    const uint64_t E = ctx->E, buckets = uint64_t(n) * n;
    if (bucket_offsets[0] != 0 || bucket_offsets[buckets] != E)
      throw std::invalid_argument("bucket offsets do not cover the edge list");
    DeviceGuard g(ctx->device);
    std::vector<uint32_t> o(E);
    for (uint64_t i = 0; i < E; ++i) {
      if (edge_order[i] >= E) throw std::invalid_argument("edge order index out of range");
      o[i] = (uint32_t)edge_order[i];
    }
    DevBuf<uint32_t> order;
    order.reserve(std::max<uint64_t>(E, 1));
    LGD_CUDA(cudaMemcpy(order.get(), o.data(), E * 4, cudaMemcpyHostToDevice));
    ctx->edges_bucketed.reserve(std::max<uint64_t>(E * 3, 3));
    launch_gather_u32x3(ctx->edges.get(), order.get(), E, ctx->edges_bucketed.get(), ctx->stream);
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->offsets.assign(bucket_offsets, bucket_offsets + buckets + 1);
    ctx->n = n;
    ctx->stride = (ctx->V + n - 1) / n;
    ctx->partitioned = true;
    if (n <= 3) {
      ctx->plan = single_state_plan(n);
      ctx->planned = true;
    } else if (!ctx->planned || ctx->plan.seq.n != n) {
      ctx->plan = make_iteration_plan(make_loading_order(n), n);
      ctx->planned = true;
    }
  });
}

int lgd_plan_iteration_order(uint32_t n, uint64_t capacity, uint64_t* num_states,
                             uint32_t* states, uint32_t* swaps, uint32_t* bucket_order,
                             uint64_t* state_offsets, uint64_t* prefetch_points) {
  return guarded([&] {
    const IterationPlan plan = make_iteration_plan(make_loading_order(n), n);
    const uint64_t S = plan.seq.states.size();
    if (num_states) *num_states = S;
    if (capacity < S) return;
    for (uint64_t i = 0; i < S; ++i)
      for (int j = 0; j < 3; ++j) states[3 * i + j] = plan.seq.states[i][j];
    for (uint64_t i = 0; i + 1 < S; ++i) {
      swaps[2 * i] = plan.seq.swaps[i].evicted;
      swaps[2 * i + 1] = plan.seq.swaps[i].loaded;
    }
    for (size_t g = 0; g < plan.bucket_order.size(); ++g) {
      bucket_order[2 * g] = plan.bucket_order[g].first;
      bucket_order[2 * g + 1] = plan.bucket_order[g].second;
    }
    std::memcpy(state_offsets, plan.state_offsets.data(), (S + 1) * 8);
    if (S > 1) std::memcpy(prefetch_points, plan.prefetch_points.data(), (S - 1) * 8);
  });
}

int lgd_set_iteration_plan(lgd_context* ctx, uint64_t num_states, const uint32_t* states,
                           const uint32_t* swaps, const uint32_t* bucket_order,
                           const uint64_t* state_offsets, const uint64_t* prefetch_points) {
  return guarded([&] {
    if (!ctx || !states || !bucket_order || !state_offsets)
      throw std::invalid_argument("null argument");
    if (!ctx->partitioned) throw std::invalid_argument("set a partition plan first");
    const uint32_t n = ctx->n;
    if (num_states == 0) throw std::invalid_argument("plan needs at least one state");
    IterationPlan plan;
    plan.seq.n = n;
    for (uint64_t i = 0; i < num_states; ++i) {
      std::array<uint32_t, 3> s{states[3 * i], states[3 * i + 1], states[3 * i + 2]};
      for (uint32_t p : s)
        if (p != kNoPartition && p >= n) throw std::invalid_argument("state partition out of range");
      plan.seq.states.push_back(s);
    }
    for (uint64_t i = 0; i + 1 < num_states && swaps; ++i)
      plan.seq.swaps.push_back({swaps[2 * i], swaps[2 * i + 1]});
    std::vector<uint8_t> seen(uint64_t(n) * n, 0);
    for (uint64_t g = 0; g < uint64_t(n) * n; ++g) {
      const uint32_t a = bucket_order[2 * g], b = bucket_order[2 * g + 1];
      if (a >= n || b >= n) throw std::invalid_argument("bucket id out of range");
      if (seen[uint64_t(a) * n + b]++) throw std::invalid_argument("duplicate bucket in order");
      plan.bucket_order.push_back({a, b});
    }
    plan.state_offsets.assign(state_offsets, state_offsets + num_states + 1);
    if (plan.state_offsets.front() != 0 || plan.state_offsets.back() != uint64_t(n) * n)
      throw std::invalid_argument("state offsets inconsistent with bucket order");
    if (prefetch_points && num_states > 1)
      plan.prefetch_points.assign(prefetch_points, prefetch_points + num_states - 1);
    // every bucket must be computable inside its state (ordering.cpp:371-381)
    for (uint64_t s = 0; s < num_states; ++s) {
      for (uint64_t g = plan.state_offsets[s]; g < plan.state_offsets[s + 1]; ++g) {
        const auto [a, b] = plan.bucket_order[g];
        const auto& st = plan.seq.states[s];
        auto holds = [&](uint32_t p) { return st[0] == p || st[1] == p || st[2] == p; };
        if (!holds(a) || !holds(b))
          throw std::invalid_argument("bucket scheduled while a partition is not resident");
      }
    }
    ctx->plan = std::move(plan);
    ctx->planned = true;
  });
}

int lgd_init_store(lgd_context* ctx, uint64_t seed) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (!ctx->partitioned) throw std::invalid_argument("set a partition plan first");
    DeviceGuard g(ctx->device);
    ctx->wait_stores();  // its copies do not run on the training stream
    const uint64_t V = ctx->V, d = ctx->dim;
    ctx->theta.reserve(V * d);
    ctx->state.reserve(V * d);
    ctx->rel_theta.reserve(std::max<uint64_t>(ctx->R, 1) * d);
    ctx->rel_state.reserve(std::max<uint64_t>(ctx->R, 1) * d);
    const uint64_t* J = jump_tables(ctx->device);
    for (uint32_t p = 0; p < ctx->n; ++p) {  // store.cpp:74-80
      const uint64_t rows = ctx->part_rows(p);
      launch_init_uniform(J, derive_seed(seed, p), rows * d, ctx->dim,
                          ctx->theta.get() + ctx->part_begin(p) * d, ctx->stream);
    }
    LGD_CUDA(cudaMemsetAsync(ctx->state.get(), 0, V * d * 4, ctx->stream));
    if (ctx->R) {  // store.cpp:81-86
      launch_init_uniform(J, derive_seed(seed, kTagRelations), ctx->R * d, ctx->dim,
                          ctx->rel_theta.get(), ctx->stream);
      LGD_CUDA(cudaMemsetAsync(ctx->rel_state.get(), 0, ctx->R * d * 4, ctx->stream));
    }
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->tables_ready = true;
  });
}

static void ensure_tables(lgd_context* ctx) {
  if (ctx->theta.n >= ctx->V * ctx->dim) return;
  ctx->theta.reserve(ctx->V * ctx->dim);
  ctx->state.reserve(ctx->V * ctx->dim);
  ctx->rel_theta.reserve(std::max<uint64_t>(ctx->R, 1) * ctx->dim);
  ctx->rel_state.reserve(std::max<uint64_t>(ctx->R, 1) * ctx->dim);
  LGD_CUDA(cudaMemset(ctx->theta.get(), 0, ctx->theta.bytes()));
  LGD_CUDA(cudaMemset(ctx->state.get(), 0, ctx->state.bytes()));
}

int lgd_load_partition(lgd_context* ctx, uint32_t p, const float* e_s, uint64_t rows) {
  return guarded([&] {
    if (!ctx || !e_s) throw std::invalid_argument("null argument");
    if (!ctx->partitioned || p >= ctx->n) throw std::invalid_argument("partition out of range");
    if (rows != ctx->part_rows(p)) throw std::invalid_argument("partition row count mismatch");
    DeviceGuard g(ctx->device);
    ctx->wait_stores();  // its copies do not run on the training stream
    ensure_tables(ctx);
    const uint64_t off = ctx->part_begin(p) * ctx->dim, cnt = rows * ctx->dim;
    LGD_CUDA(cudaMemcpyAsync(ctx->theta.get() + off, e_s, cnt * 4, cudaMemcpyHostToDevice,
                             ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(ctx->state.get() + off, e_s + cnt, cnt * 4, cudaMemcpyHostToDevice,
                             ctx->stream));
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->tables_ready = true;
  });
}

int lgd_store_partition(lgd_context* ctx, uint32_t p, float* e_s, uint64_t rows) {
  return guarded([&] {
    if (!ctx || !e_s) throw std::invalid_argument("null argument");
    if (!ctx->partitioned || p >= ctx->n) throw std::invalid_argument("partition out of range");
    if (rows != ctx->part_rows(p)) throw std::invalid_argument("partition row count mismatch");
    if (!ctx->tables_ready) throw std::invalid_argument("embedding store not initialised");
    DeviceGuard g(ctx->device);
    const uint64_t off = ctx->part_begin(p) * ctx->dim, cnt = rows * ctx->dim;
    LGD_CUDA(cudaMemcpyAsync(e_s, ctx->theta.get() + off, cnt * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(e_s + cnt, ctx->state.get() + off, cnt * 4, cudaMemcpyDeviceToHost,
                             ctx->stream));
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

int lgd_store_partition_async(lgd_context* ctx, uint32_t p, float* e_s, uint64_t rows) {
  return guarded([&] {
    if (!ctx || !e_s) throw std::invalid_argument("null argument");
    if (!ctx->partitioned || p >= ctx->n) throw std::invalid_argument("partition out of range");
    if (rows != ctx->part_rows(p)) throw std::invalid_argument("partition row count mismatch");
    if (!ctx->tables_ready) throw std::invalid_argument("embedding store not initialised");
    DeviceGuard g(ctx->device);
    if (!ctx->store_stream) {
      LGD_CUDA(cudaStreamCreateWithFlags(&ctx->store_stream, cudaStreamNonBlocking));
      LGD_CUDA(cudaEventCreateWithFlags(&ctx->ev_store_src, cudaEventDisableTiming));
      LGD_CUDA(cudaEventCreateWithFlags(&ctx->ev_store_done, cudaEventDisableTiming));
    }
    // the partition as the training stream's work so far leaves it
    LGD_CUDA(cudaEventRecord(ctx->ev_store_src, ctx->stream));
    LGD_CUDA(cudaStreamWaitEvent(ctx->store_stream, ctx->ev_store_src, 0));
    const uint64_t off = ctx->part_begin(p) * ctx->dim, cnt = rows * ctx->dim;
    LGD_CUDA(cudaMemcpyAsync(e_s, ctx->theta.get() + off, cnt * 4, cudaMemcpyDeviceToHost,
                             ctx->store_stream));
    LGD_CUDA(cudaMemcpyAsync(e_s + cnt, ctx->state.get() + off, cnt * 4, cudaMemcpyDeviceToHost,
                             ctx->store_stream));
    LGD_CUDA(cudaEventRecord(ctx->ev_store_done, ctx->store_stream));
    ctx->stores_pending = true;
  });
}

int lgd_wait_stores(lgd_context* ctx) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->wait_stores();
  });
}

int lgd_set_relations(lgd_context* ctx, const float* e_s, uint64_t count) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (count != ctx->R) throw std::invalid_argument("relation count mismatch");
    if (!count) return;
    DeviceGuard g(ctx->device);
    ctx->wait_stores();  // its copies do not run on the training stream
    ensure_tables(ctx);
    const uint64_t cnt = count * ctx->dim;
    LGD_CUDA(cudaMemcpy(ctx->rel_theta.get(), e_s, cnt * 4, cudaMemcpyHostToDevice));
    LGD_CUDA(cudaMemcpy(ctx->rel_state.get(), e_s + cnt, cnt * 4, cudaMemcpyHostToDevice));
  });
}

int lgd_get_relations(lgd_context* ctx, float* e_s, uint64_t count) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (count != ctx->R) throw std::invalid_argument("relation count mismatch");
    if (!count) return;
    DeviceGuard g(ctx->device);
    const uint64_t cnt = count * ctx->dim;
    LGD_CUDA(cudaMemcpy(e_s, ctx->rel_theta.get(), cnt * 4, cudaMemcpyDeviceToHost));
    LGD_CUDA(cudaMemcpy(e_s + cnt, ctx->rel_state.get(), cnt * 4, cudaMemcpyDeviceToHost));
  });
}

int lgd_train_epoch(lgd_context* ctx, uint32_t epoch, lgd_epoch_result* out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->train_range(epoch, 0, ctx->plan.bucket_order.size(), out);
  });
}

int lgd_train_buckets(lgd_context* ctx, uint32_t epoch, uint64_t g_begin, uint64_t g_end,
                      lgd_epoch_result* out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->train_range(epoch, g_begin, g_end, out);
  });
}

int lgd_train_bucket_prefix(lgd_context* ctx, uint32_t epoch, uint64_t g, uint64_t max_batches,
                            double* batch_losses, uint64_t* batch_nodes, lgd_epoch_result* out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard dg(ctx->device);
    ctx->fence_stores();
    ctx->check_ready();
    if (g >= ctx->plan.bucket_order.size()) throw std::invalid_argument("bucket position out of range");
    const uint64_t limit = max_batches ? max_batches : ~uint64_t(0);
    const auto items = ctx->plan_items(g, g + 1);
    const uint64_t m = ctx->bucket_size(items[0]);
    const uint64_t nb = std::min<uint64_t>(limit, (m + ctx->opt.batch_size - 1) / ctx->opt.batch_size);
    DevBuf<unsigned long long> trace;
    trace.reserve(std::max<uint64_t>(nb, 1));
    ctx->train_items(epoch, items, out, ctx->host_edges, limit, batch_nodes ? trace.get() : nullptr);
    if (batch_losses && nb)
      LGD_CUDA(cudaMemcpy(batch_losses, ctx->batch_losses.get(), nb * 8, cudaMemcpyDeviceToHost));
    if (batch_nodes && nb) {
      std::vector<unsigned long long> c(nb);
      LGD_CUDA(cudaMemcpy(c.data(), trace.get(), nb * 8, cudaMemcpyDeviceToHost));
      for (uint64_t b = 0; b < nb; ++b) batch_nodes[b] = c[b] - (b ? c[b - 1] : 0);
    }
  });
}

int lgd_round_schedule(uint32_t n, uint64_t capacity, uint64_t* count, lgd_bucket_item* items,
                       uint32_t* num_rounds, uint32_t* pairs_per_round) {
  return guarded([&] {
    const RoundSchedule rs = make_round_schedule(n);
    if (count) *count = rs.buckets.size();
    if (num_rounds) *num_rounds = rs.num_rounds;
    if (pairs_per_round) *pairs_per_round = rs.pairs_per_round;
    if (capacity < rs.buckets.size() || !items) return;
    for (size_t i = 0; i < rs.buckets.size(); ++i) {
      const auto& b = rs.buckets[i];
      items[i] = lgd_bucket_item{b.src, b.dst, b.g, {b.pool[0], b.pool[1], kNoPartition},
                                 b.round, b.pair};
    }
  });
}

static std::vector<lgd_context::WorkItem> work_items(const lgd_context* ctx,
                                                     const lgd_bucket_item* items, uint64_t count) {
  std::vector<lgd_context::WorkItem> out;
  for (uint64_t i = 0; i < count; ++i) {
    const auto& it = items[i];
    if (it.src_part >= ctx->n || it.dst_part >= ctx->n)
      throw std::invalid_argument("bucket partition out of range");
    const Pool pool = ctx->pool_of_parts(it.pool, 3);
    // both endpoints of the bucket must be in its pool (resident)
    auto in_pool = [&](uint32_t p) {
      return it.pool[0] == p || it.pool[1] == p || it.pool[2] == p;
    };
    if (!in_pool(it.src_part) || !in_pool(it.dst_part))
      throw std::invalid_argument("bucket scheduled while a partition is not resident");
    out.push_back({it.src_part, it.dst_part, it.g, pool});
  }
  return out;
}

int lgd_train_items(lgd_context* ctx, uint32_t epoch, const lgd_bucket_item* items,
                    uint64_t count, lgd_epoch_result* out) {
  return guarded([&] {
    if (!ctx || (!items && count)) throw std::invalid_argument("null argument");
    if (!ctx->partitioned) throw std::invalid_argument("no partition plan");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->train_items(epoch, work_items(ctx, items, count), out, ctx->host_edges);
  });
}

int lgd_round_begin(lgd_context* ctx, uint32_t epoch, const lgd_bucket_item* items,
                    uint64_t count, uint64_t* my_batches) {
  return guarded([&] {
    if (!ctx || (!items && count)) throw std::invalid_argument("null argument");
    if (!ctx->partitioned) throw std::invalid_argument("no partition plan");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    const uint64_t b = ctx->round_begin(epoch, work_items(ctx, items, count));
    if (my_batches) *my_batches = b;
  });
}

int lgd_round_step(lgd_context* ctx, uint64_t step, double* rel_grad_device) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->round_step(step, rel_grad_device);
  });
}

int lgd_round_apply_relations(lgd_context* ctx, const double* summed_device) {
  return guarded([&] {
    if (!ctx || !summed_device) throw std::invalid_argument("null argument");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->round_apply_relations(summed_device);
  });
}

int lgd_get_stream(lgd_context* ctx, void** cuda_stream) {
  return guarded([&] {
    if (!ctx || !cuda_stream) throw std::invalid_argument("null argument");
    DeviceGuard g(ctx->device);
    // work the caller queues on this stream is ordered after pending
    // asynchronous write-backs, like the library's own table writes
    ctx->fence_stores();
    *cuda_stream = (void*)ctx->stream;
  });
}

int lgd_set_stream_ordered(lgd_context* ctx, int on) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    ctx->stream_ordered = on != 0;
  });
}

int lgd_round_end(lgd_context* ctx, lgd_epoch_result* out) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->round_end(out);
  });
}

int lgd_device_tables(lgd_context* ctx, float** theta, float** state, float** rel_theta,
                      float** rel_state) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    {
      DeviceGuard g(ctx->device);
      ctx->wait_stores();  // the caller may write through these on any stream
    }
    if (theta) *theta = ctx->theta.get();
    if (state) *state = ctx->state.get();
    if (rel_theta) *rel_theta = ctx->rel_theta.get();
    if (rel_state) *rel_state = ctx->rel_state.get();
  });
}

int lgd_train_buckets_from_host(lgd_context* ctx, uint32_t epoch, uint64_t g_begin,
                                uint64_t g_end, const uint32_t* host_bucketed_edges,
                                lgd_epoch_result* out) {
  return guarded([&] {
    if (!ctx || !host_bucketed_edges) throw std::invalid_argument("null argument");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->train_range(epoch, g_begin, g_end, out, host_bucketed_edges);
  });
}

int lgd_set_host_edges(lgd_context* ctx, const uint32_t* host_bucketed_edges) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    ctx->host_edges = host_bucketed_edges;
  });
}

int lgd_get_bucketed_edges(lgd_context* ctx, uint32_t* edges_out) {
  return guarded([&] {
    if (!ctx || !edges_out) throw std::invalid_argument("null argument");
    if (!ctx->partitioned) throw std::invalid_argument("no partition plan");
    DeviceGuard g(ctx->device);
    LGD_CUDA(cudaMemcpy(edges_out, ctx->edges_bucketed.get(), ctx->E * 12,
                        cudaMemcpyDeviceToHost));
  });
}

int lgd_host_alloc(uint64_t bytes, void** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null argument");
    LGD_CUDA(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable));
  });
}

int lgd_host_free(void* p) {
  return guarded([&] {
    if (p) LGD_CUDA(cudaFreeHost(p));
  });
}

int lgd_train_batch(lgd_context* ctx, const uint32_t* edges, uint64_t num_positives,
                    const uint32_t* negatives, int apply, double* loss, uint64_t* unique_nodes,
                    uint64_t* unique_rels) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->upload_batch(edges, num_positives, negatives);
    LGD_CUDA(cudaMemsetAsync(ctx->counters.get(), 0, 16, ctx->stream));
    LGD_CUDA(cudaMemsetAsync(ctx->batch_losses.get(), 0, 8, ctx->stream));
    DevBuf<double> gn, gr;
    DevBuf<uint8_t> fn, fr;
    if (!apply) {  // loss + unique counts only: route gradients to scratch
      gn.reserve(ctx->V * ctx->dim);
      fn.reserve(ctx->V);
      gr.reserve(std::max<uint64_t>(ctx->R, 1) * ctx->dim);
      fr.reserve(std::max<uint64_t>(ctx->R, 1));
    }
    BatchArgs a = ctx->batch_args(ctx->op_edges.get(), ctx->op_negs.get(), num_positives,
                                  ctx->batch_losses.get());
    if (!apply) {
      a.grad_nodes = gn.get();
      a.grad_node_flag = fn.get();
      a.grad_rels = gr.get();
      a.grad_rel_flag = fr.get();
      a.side = nullptr;
    }
    launch_train_batch(a, ctx->stream, nullptr);
    ctx->launches += ctx->batch_launches();
    double l = 0;
    unsigned long long cnt[2];
    LGD_CUDA(cudaMemcpyAsync(&l, ctx->batch_losses.get(), 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(cnt, ctx->counters.get(), 16, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (loss) *loss = l;
    if (unique_nodes) *unique_nodes = cnt[0];
    if (unique_rels) *unique_rels = cnt[1];
  });
}

int lgd_batch_gradients(lgd_context* ctx, const uint32_t* edges, uint64_t num_positives,
                        const uint32_t* negatives, double* loss, uint64_t* num_nodes,
                        uint32_t* node_ids, double* node_grads, uint64_t* num_rels,
                        uint32_t* rel_ids, double* rel_grads) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    ctx->upload_batch(edges, num_positives, negatives);
    const uint64_t V = ctx->V, R = std::max<uint64_t>(ctx->R, 1), d = ctx->dim;
    DevBuf<double> gn, gr;
    DevBuf<uint8_t> fn, fr;
    gn.reserve(V * d);
    fn.reserve(V);
    gr.reserve(R * d);
    fr.reserve(R);
    LGD_CUDA(cudaMemsetAsync(fn.get(), 0, V, ctx->stream));
    LGD_CUDA(cudaMemsetAsync(fr.get(), 0, R, ctx->stream));
    LGD_CUDA(cudaMemsetAsync(ctx->counters.get(), 0, 16, ctx->stream));
    BatchArgs a = ctx->batch_args(ctx->op_edges.get(), ctx->op_negs.get(), num_positives,
                                  ctx->batch_losses.get());
    a.grad_nodes = gn.get();
    a.grad_node_flag = fn.get();
    a.grad_rels = gr.get();
    a.grad_rel_flag = fr.get();
    a.side = nullptr;
    launch_train_batch(a, ctx->stream, nullptr);
    std::vector<uint8_t> hf(V), hrf(R);
    std::vector<double> hg(V * d), hr(R * d);
    double l = 0;
    LGD_CUDA(cudaMemcpyAsync(&l, ctx->batch_losses.get(), 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(hf.data(), fn.get(), V, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(hg.data(), gn.get(), V * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(hrf.data(), fr.get(), R, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(hr.data(), gr.get(), R * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (loss) *loss = l;
    uint64_t u = 0;
    for (uint64_t v = 0; v < V; ++v) {
      if (!hf[v]) continue;
      if (node_ids) node_ids[u] = (uint32_t)v;
      if (node_grads) std::memcpy(node_grads + u * d, hg.data() + v * d, d * 8);
      ++u;
    }
    if (num_nodes) *num_nodes = u;
    uint64_t ur = 0;
    if (ctx->typed()) {
      for (uint64_t r = 0; r < ctx->R; ++r) {
        if (!hrf[r]) continue;
        if (rel_ids) rel_ids[ur] = (uint32_t)r;
        if (rel_grads) std::memcpy(rel_grads + ur * d, hr.data() + r * d, d * 8);
        ++ur;
      }
    }
    if (num_rels) *num_rels = ur;
  });
}

int lgd_evaluate(lgd_context* ctx, const uint32_t* test_edges, uint64_t count,
                 uint32_t num_candidates, uint32_t hits_k, uint64_t seed, double* mrr,
                 double* hits_at_k) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (count == 0) throw std::invalid_argument("test edge set is empty");
    if (num_candidates == 0) throw std::invalid_argument("need at least one candidate");
    if (!ctx->tables_ready) throw std::invalid_argument("embedding store not initialised");
    for (uint64_t t = 0; t < count; ++t) {
      const uint32_t s = test_edges[3 * t], r = test_edges[3 * t + 1], d = test_edges[3 * t + 2];
      if (ctx->typed() && r == LGD_NO_RELATION)
        throw std::invalid_argument("typed model requires a relation id on every edge");
      if (ctx->typed() && r >= ctx->R) throw std::out_of_range("relation id out of range");
      if (s >= ctx->V || d >= ctx->V) throw std::out_of_range("node is not resident");
    }
    DeviceGuard g(ctx->device);
    if (eval_smem_bytes(ctx->dim) > 227 * 1024) throw std::invalid_argument("dimension too large for evaluate");
    // candidates in tiles of test edges: scratch <= 256 MB whatever the count
    const uint64_t tile = std::max<uint64_t>(1, std::min<uint64_t>(count, (64ull << 20) / num_candidates));
    DevBuf<uint32_t> dedges, cand;
    DevBuf<double> rr, hit;
    dedges.reserve(count * 3);
    cand.reserve(tile * num_candidates);
    rr.reserve(count);
    hit.reserve(count);
    LGD_CUDA(cudaMemcpyAsync(dedges.get(), test_edges, count * 12, cudaMemcpyHostToDevice,
                             ctx->stream));
    EvalArgs a{ctx->kind, ctx->dim, ctx->theta.get(), ctx->rel_theta.get(), dedges.get(), count,
               num_candidates, hits_k, ctx->V, seed, cand.get(), rr.get(), hit.get()};
    if (ctx->profiling) LGD_CUDA(cudaEventRecord(ctx->ev_begin, ctx->stream));
    for (uint64_t t0 = 0; t0 < count; t0 += tile) {
      launch_evaluate_tile(a, t0, std::min(tile, count - t0), ctx->stream);
      ctx->launches += 2;
    }
    if (ctx->profiling) LGD_CUDA(cudaEventRecord(ctx->ev_end, ctx->stream));
    std::vector<double> hr(count), hh(count);
    LGD_CUDA(cudaMemcpyAsync(hr.data(), rr.get(), count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaMemcpyAsync(hh.data(), hit.get(), count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->profiling) {
      float ms = 0;
      LGD_CUDA(cudaEventElapsedTime(&ms, ctx->ev_begin, ctx->ev_end));
      ctx->eval_ms = ms;
    }
    // result.mrr / hits_at_k accumulate in edge order, then / edges (train.cpp:406-411)
    double m = 0.0, hk = 0.0;
    for (uint64_t t = 0; t < count; ++t) {
      m += hr[t];
      hk += hh[t];
    }
    if (mrr) *mrr = m / (double)count;
    if (hits_at_k) *hits_at_k = hk / (double)count;
  });
}

// ------------------------------------------------- sampler primitives
static void primitive_setup(int device, uint64_t seed, uint64_t skip, DevBuf<uint64_t>& pos,
                            DevBuf<unsigned long long>& rej, StreamSlot& slot) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    throw lgd::cuda_error("no CUDA device: the B200 path has no CPU fallback");
  if (device < 0 || device >= count) throw std::invalid_argument("bad device ordinal");
  pos.reserve(1);
  rej.reserve(1);
  LGD_CUDA(cudaMemcpy(pos.get(), &skip, 8, cudaMemcpyHostToDevice));
  LGD_CUDA(cudaMemset(rej.get(), 0xff, 8));
  slot.origin = xo_seed(seed);
  slot.d_pos = pos.get();
  slot.d_reject = rej.get();
  jump_tables(device);
}

int lgd_rng_below(int device, uint64_t seed, uint64_t skip, uint64_t bound, uint64_t count,
                  uint64_t* out, uint64_t* consumed) {
  return guarded([&] {
    if (bound == 0) throw std::invalid_argument("bound must be positive");
    DeviceGuard g(device);
    DevBuf<uint64_t> pos, o;
    DevBuf<unsigned long long> rej;
    StreamSlot slot{};
    primitive_setup(device, seed, skip, pos, rej, slot);
    o.reserve(std::max<uint64_t>(count, 1));
    launch_below_u64(slot, count, bound, o.get(), nullptr);
    uint64_t p = 0;
    LGD_CUDA(cudaMemcpy(&p, pos.get(), 8, cudaMemcpyDeviceToHost));
    if (count) LGD_CUDA(cudaMemcpy(out, o.get(), count * 8, cudaMemcpyDeviceToHost));
    if (consumed) *consumed = p - skip;
  });
}

int lgd_sample_negatives(int device, uint64_t seed, uint64_t skip, const uint64_t* first,
                         const uint64_t* counts, int num_ranges, uint32_t k,
                         uint64_t num_positives, uint32_t* out, uint64_t* consumed) {
  return guarded([&] {
    if (k == 0) throw std::invalid_argument("at least one negative per positive required");
    if (num_ranges < 1 || num_ranges > 3) throw std::invalid_argument("1 to 3 resident ranges");
    DeviceGuard g(device);
    Pool pool{};
    uint64_t acc = 0;
    for (int i = 0; i < num_ranges; ++i) {
      pool.first[i] = first[i];
      acc += counts[i];
      pool.end_index[i] = acc;
    }
    pool.n = num_ranges;
    if (acc == 0) throw std::invalid_argument("no resident nodes to sample from");
    DevBuf<uint64_t> pos;
    DevBuf<uint32_t> o;
    DevBuf<unsigned long long> rej;
    StreamSlot slot{};
    primitive_setup(device, seed, skip, pos, rej, slot);
    const uint64_t n = num_positives * k;
    o.reserve(std::max<uint64_t>(n, 1));
    launch_sample_nodes(slot, n, pool, o.get(), nullptr);
    uint64_t p = 0;
    LGD_CUDA(cudaMemcpy(&p, pos.get(), 8, cudaMemcpyDeviceToHost));
    if (n) LGD_CUDA(cudaMemcpy(out, o.get(), n * 4, cudaMemcpyDeviceToHost));
    if (consumed) *consumed = p - skip;
  });
}

int lgd_shuffle_permutation(int device, uint64_t seed, uint64_t m, uint32_t* perm,
                            uint64_t* consumed) {
  return guarded([&] {
    if (m >= 0xffffffffull) throw std::invalid_argument("bucket too large");
    DeviceGuard g(device);
    DevBuf<uint64_t> pos;
    DevBuf<unsigned long long> rej;
    StreamSlot slot{};
    primitive_setup(device, seed, 0, pos, rej, slot);
    if (m == 0) {
      if (consumed) *consumed = 0;
      return;
    }
    DevBuf<uint32_t> H, P, ki, vi, ko, vo, ptr, G;
    DevBuf<unsigned char> temp;
    for (auto* b : {&H, &P, &ki, &vi, &ko, &vo, &ptr, &G}) b->reserve(m);
    temp.reserve(shuffle_sort_temp_bytes(m));
    launch_shuffle_draws(slot, m, H.get(), nullptr);
    ShuffleScratch s{ki.get(), vi.get(), ko.get(), vo.get(), ptr.get(), G.get(), temp.get(),
                     temp.bytes()};
    launch_shuffle_permutation(H.get(), m, s, P.get(), nullptr);
    uint64_t p = 0;
    LGD_CUDA(cudaMemcpy(&p, pos.get(), 8, cudaMemcpyDeviceToHost));
    LGD_CUDA(cudaMemcpy(perm, P.get(), m * 4, cudaMemcpyDeviceToHost));
    if (consumed) *consumed = p;
  });
}

int lgd_set_profiling(lgd_context* ctx, int enabled) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    if (enabled && ctx->prof_events.empty()) {
      ctx->prof_events.resize(kProfRing * 5);
      for (auto& e : ctx->prof_events) LGD_CUDA(cudaEventCreate(&e));
      ctx->prof_pending.assign(kProfRing, 0);
    }
    if (!enabled) ctx->prof_flush();
    ctx->profiling = enabled != 0;
  });
}

int lgd_get_kernel_stats(lgd_context* ctx, int which, lgd_kernel_stats* out) {
  return guarded([&] {
    if (!ctx || !out) throw std::invalid_argument("null argument");
    if (which < 0 || which >= LGD_KSTAT_COUNT) throw std::invalid_argument("bad stat id");
    ctx->prof_flush();
    *out = ctx->kstats[which];
  });
}

int lgd_reset_kernel_stats(lgd_context* ctx) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    ctx->prof_flush();
    for (auto& s : ctx->kstats) s = lgd_kernel_stats{};
    ctx->launches = 0;
  });
}

uint64_t lgd_launch_count(lgd_context* ctx) { return ctx ? ctx->launches : 0; }

int lgd_synchronize(lgd_context* ctx) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    DeviceGuard g(ctx->device);
    LGD_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

}  // extern "C"
