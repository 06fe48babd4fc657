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

#include "context.hpp"

// ============================================================== C ABI ====
extern "C" {

const char* lgd_last_error(void) { return g_last_error.c_str(); }

// shared-negative chunks (shared.cu): 16-byte operand rows, the mix / G
// accumulators within 128 TMEM columns, the dot-product models
static void check_shared_mode(int model_kind, uint32_t dim, const lgd_train_options& o) {
  if (!o.shared_chunk) return;
  if (model_kind == LGD_MODEL_TRANSE)
    throw std::invalid_argument("shared-negative chunks support the Dot, DistMult and ComplEx models");
  if (dim % 4 != 0 || dim > 128)
    throw std::invalid_argument("shared-negative chunks need a dimension that is a multiple of 4, at most 128");
}

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
    if (options) check_shared_mode(model_kind, dim, *options);
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
      if (const char* env = std::getenv("LGD_K4")) {
        const long v = std::strtol(env, nullptr, 10);
        c->seg_rows = v != 1;
        c->k4_variant = v == 3 ? 1 : (v == 4 ? 2 : 0);
      }
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
      LGD_CUDA(cudaEventCreateWithFlags(&c->ev_long, cudaEventDisableTiming));
      LGD_CUDA(cudaEventCreateWithFlags(&c->ev_long_done, cudaEventDisableTiming));
      for (auto* e : {&c->copy_done[0], &c->copy_done[1], &c->stage_free[0], &c->stage_free[1],
                      &c->ev_prepped[0], &c->ev_prepped[1], &c->ev_consumed[0], &c->ev_consumed[1]})
        LGD_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
      // the next bucket's prep (opt-in): lowest priority, so the batches on
      // the training stream (the critical path) are scheduled first
      if (const char* env = std::getenv("LGD_OVERLAP_PREP"))
        c->overlap_prep = std::strtol(env, nullptr, 10) != 0;
      if (c->overlap_prep) {
        int lo = 0, hi = 0;
        LGD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        LGD_CUDA(cudaStreamCreateWithPriority(&c->prep_stream, cudaStreamNonBlocking, lo));
      }
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
    check_shared_mode(ctx->kind, ctx->dim, *options);
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

// batch_gradients (train.cpp:280-340) as a GradientSet.  Exact path with
// vector-lane dims: compact -- the sorted segment heads give the unique ids,
// one warp per segment writes its FP64 row (O(unique rows) memory, ids
// ascending like the reference's std::map).  Shared-negative chunks and the
// 8-lane-group dims keep the dense scratch route.
static void compact_gradients(lgd_context* ctx, uint64_t P, double* loss, uint64_t* num_nodes,
                              uint32_t* node_ids, double* node_grads, uint64_t* num_rels,
                              uint32_t* rel_ids, double* rel_grads) {
  const uint64_t d = ctx->dim, n = P * (ctx->k() + 2);
  DevBuf<uint32_t> seg, rseg, rk, rv, cnt;
  DevBuf<unsigned char> temp;
  seg.reserve(n + 1);
  cnt.reserve(2);
  const bool typed = ctx->typed() && ctx->R;
  if (typed) {
    rseg.reserve(P + 1);
    rk.reserve(P);
    rv.reserve(P);
  }
  temp.reserve(grads_select_temp_bytes(n));
  LGD_CUDA(cudaMemsetAsync(cnt.get(), 0, 8, ctx->stream));
  GradCompact gc{seg.get(), typed ? rseg.get() : nullptr, rk.get(), rv.get(), cnt.get(),
                 temp.get(), temp.bytes()};
  BatchArgs a = ctx->batch_args(ctx->op_edges.get(), ctx->op_negs.get(), P, ctx->batch_losses.get());
  a.side = nullptr;
  a.gc = &gc;
  launch_train_batch(a, ctx->stream, nullptr);
  uint32_t c[2];
  double l = 0;
  LGD_CUDA(cudaMemcpyAsync(c, cnt.get(), 8, cudaMemcpyDeviceToHost, ctx->stream));
  LGD_CUDA(cudaMemcpyAsync(&l, ctx->batch_losses.get(), 8, cudaMemcpyDeviceToHost, ctx->stream));
  LGD_CUDA(cudaStreamSynchronize(ctx->stream));
  const uint64_t nn = c[0], nr = typed ? c[1] : 0;
  if (loss) *loss = l;
  if (num_nodes) *num_nodes = nn;
  if (num_rels) *num_rels = nr;
  if (!node_ids && !node_grads && !rel_ids && !rel_grads) return;  // counts only
  DevBuf<uint32_t> ni, ri;
  DevBuf<double> ng, rg;
  ni.reserve(std::max<uint64_t>(nn, 1));
  ng.reserve(std::max<uint64_t>(nn, 1) * d);
  ri.reserve(std::max<uint64_t>(nr, 1));
  rg.reserve(std::max<uint64_t>(nr, 1) * d);
  launch_grads_phase2(a, nn, nr, ni.get(), ng.get(), ri.get(), rg.get(), ctx->stream);
  if (node_ids && nn)
    LGD_CUDA(cudaMemcpyAsync(node_ids, ni.get(), nn * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (node_grads && nn)
    LGD_CUDA(cudaMemcpyAsync(node_grads, ng.get(), nn * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (rel_ids && nr)
    LGD_CUDA(cudaMemcpyAsync(rel_ids, ri.get(), nr * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (rel_grads && nr)
    LGD_CUDA(cudaMemcpyAsync(rel_grads, rg.get(), nr * d * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LGD_CUDA(cudaStreamSynchronize(ctx->stream));
}

static bool compact_ok(const lgd_context* ctx) {
  return !ctx->chunk() && k4_vec_width(ctx->kind, ctx->dim) != 0;
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
    if (!apply && compact_ok(ctx)) {  // loss + unique counts: the segment heads, no scratch rows
      compact_gradients(ctx, num_positives, loss, unique_nodes, nullptr, nullptr, unique_rels,
                        nullptr, nullptr);
      return;
    }
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
    if (compact_ok(ctx)) {
      compact_gradients(ctx, num_positives, loss, num_nodes, node_ids, node_grads, num_rels,
                        rel_ids, rel_grads);
      return;
    }
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
    if (ctx->profiling) {  // K6: (candidates + 1 + typed) rows and the edge record per test edge
      float ms = 0;
      LGD_CUDA(cudaEventElapsedTime(&ms, ctx->ev_begin, ctx->ev_end));
      auto& ks = ctx->kstats[LGD_KSTAT_EVAL];
      ks.launches += 1;
      ks.total_ms += ms;
      ks.algorithmic_bytes += double(count) * (12.0 + 4.0 * ctx->dim *
                                               (num_candidates + 2.0 + (ctx->typed() ? 1 : 0)));
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
