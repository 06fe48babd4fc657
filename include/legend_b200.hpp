// legend_b200.hpp -- header-only C++ face of the C ABI in legend_b200.h,
// shaped like the reference trainer's API (legend::run_epoch, batch_loss /
// batch_gradients / adagrad_step, evaluate; proj/include/legend/*.hpp) and
// throwing the same exception classes:
//   LGD_INVALID_ARGUMENT -> std::invalid_argument
//   LGD_LOGIC_ERROR      -> std::logic_error
//   LGD_OUT_OF_RANGE     -> std::out_of_range
//   LGD_RUNTIME_ERROR    -> std::runtime_error
// Link with -llegend_b200 (paper_2505_09258_b200/liblegend_b200.so).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "legend_b200.h"

namespace legend_b200 {

inline void check(int rc) {
  if (rc == LGD_OK) return;
  const std::string msg = lgd_last_error();
  switch (rc) {
    case LGD_INVALID_ARGUMENT:
      throw std::invalid_argument(msg);
    case LGD_LOGIC_ERROR:
      throw std::logic_error(msg);
    case LGD_OUT_OF_RANGE:
      throw std::out_of_range(msg);
    default:
      throw std::runtime_error(msg);
  }
}

enum class ScoreKind {
  kDot = LGD_MODEL_DOT,
  kDistMult = LGD_MODEL_DISTMULT,
  kComplEx = LGD_MODEL_COMPLEX,
  kTransE = LGD_MODEL_TRANSE  // not in the reference (parity vs the restatement)
};

struct ScoreModel {  // train.hpp:15-23
  ScoreKind kind = ScoreKind::kDot;
  std::uint32_t dim = 0;
};

struct TrainOptions {  // pipeline.hpp:89-97 (+ AdagradHyper, train.hpp:109-112)
  double learning_rate = 0.1;
  double adagrad_epsilon = 1e-10;
  std::uint32_t batch_size = 100000;
  std::uint32_t negatives = 16;
  bool shuffle = true;
  std::uint64_t seed = 0;
  // 0: the reference's per-positive negatives; C > 0: shared-negative chunks
  // (lgd_train_options.shared_chunk; last, so reference-shaped aggregate
  // initialisers keep their meaning)
  std::uint32_t shared_chunk = 0;
  lgd_train_options c() const {
    return lgd_train_options{learning_rate, adagrad_epsilon, batch_size, negatives,
                             shuffle ? 1 : 0, shared_chunk, seed};
  }
};

using EpochResult = lgd_epoch_result;  // pipeline.hpp:99-107 + device accounting

struct EvalResult {  // train.hpp:129-133
  double mrr = 0.0;
  double hits_at_k = 0.0;
};

// One HBM-resident training context: graph, partition plan, iteration plan,
// E||S tables.  Move-only.
class Trainer {
 public:
  Trainer(ScoreModel model, TrainOptions options, int device = 0) : model_(model) {
    const lgd_train_options o = options.c();
    check(lgd_create(&ctx_, static_cast<int>(model.kind), model.dim, &o, device));
  }
  ~Trainer() {
    if (ctx_) lgd_destroy(ctx_);
  }
  Trainer(const Trainer&) = delete;
  Trainer& operator=(const Trainer&) = delete;
  Trainer(Trainer&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)), model_(o.model_) {}

  // Graph: edges as (src, rel, dst) u32 triples (graph.hpp:19-25).
  void set_graph(const std::vector<std::uint32_t>& edges, std::uint64_t num_nodes,
                 std::uint64_t num_relations) {
    check(lgd_set_graph(ctx_, edges.data(), edges.size() / 3, num_nodes, num_relations));
  }
  // make_partition_plan (graph.cpp:120-150); returns bucket_offsets.  The
  // reference iteration plan is attached automatically (n >= 4).
  std::vector<std::uint64_t> make_partition_plan(std::uint32_t n) {
    std::vector<std::uint64_t> offsets(std::size_t(n) * n + 1);
    check(lgd_make_partition_plan(ctx_, n, offsets.data(), nullptr));
    return offsets;
  }
  void set_partition_plan(std::uint32_t n, const std::vector<std::uint64_t>& bucket_offsets,
                          const std::vector<std::uint64_t>& edge_order) {
    check(lgd_set_partition_plan(ctx_, n, bucket_offsets.data(), edge_order.data()));
  }
  // IterationPlan (ordering.hpp:40-47) as flat arrays.
  void set_iteration_plan(const std::vector<std::uint32_t>& states,
                          const std::vector<std::uint32_t>& swaps,
                          const std::vector<std::uint32_t>& bucket_order,
                          const std::vector<std::uint64_t>& state_offsets,
                          const std::vector<std::uint64_t>& prefetch_points) {
    check(lgd_set_iteration_plan(ctx_, states.size() / 3, states.data(),
                                 swaps.empty() ? nullptr : swaps.data(), bucket_order.data(),
                                 state_offsets.data(),
                                 prefetch_points.empty() ? nullptr : prefetch_points.data()));
  }
  void init_store(std::uint64_t seed) { check(lgd_init_store(ctx_, seed)); }
  // E||S blob of partition p (store.hpp:14-33).
  void load_partition(std::uint32_t p, const std::vector<float>& e_s) {
    check(lgd_load_partition(ctx_, p, e_s.data(), e_s.size() / (2 * model_.dim)));
  }
  std::vector<float> store_partition(std::uint32_t p, std::uint64_t rows) {
    std::vector<float> out(2 * rows * model_.dim);
    check(lgd_store_partition(ctx_, p, out.data(), rows));
    return out;
  }
  void set_relations(const std::vector<float>& e_s) {
    check(lgd_set_relations(ctx_, e_s.data(), e_s.size() / (2 * model_.dim)));
  }
  std::vector<float> get_relations(std::uint64_t count) {
    std::vector<float> out(2 * count * model_.dim);
    check(lgd_get_relations(ctx_, out.data(), count));
    return out;
  }

  // run_epoch real-train (pipeline.cpp:273-322).
  EpochResult run_epoch(std::uint32_t epoch) {
    EpochResult r{};
    check(lgd_train_epoch(ctx_, epoch, &r));
    return r;
  }
  // batch_loss + batch_gradients + adagrad_step (train.cpp:217-363); returns the loss.
  double train_batch(const std::vector<std::uint32_t>& positives,
                     const std::vector<std::uint32_t>& negatives, bool apply = true) {
    double loss = 0.0;
    check(lgd_train_batch(ctx_, positives.data(), positives.size() / 3, negatives.data(),
                          apply ? 1 : 0, &loss, nullptr, nullptr));
    return loss;
  }
  // evaluate (train.cpp:375-412).
  EvalResult evaluate(const std::vector<std::uint32_t>& test_edges, std::uint32_t num_candidates,
                      std::uint32_t hits_k, std::uint64_t seed) {
    EvalResult r;
    check(lgd_evaluate(ctx_, test_edges.data(), test_edges.size() / 3, num_candidates, hits_k, seed,
                       &r.mrr, &r.hits_at_k));
    return r;
  }

  // ---- multi-GPU partition rounds (rounds.cu; one process per GPU) ----
  // id: 128 bytes from comm_unique_id() on rank 0, shared with every rank
  void comm_init(const void* nccl_id, std::uint32_t rank, std::uint32_t world) {
    check(lgd_comm_init(ctx_, nccl_id, rank, world));
  }
  std::uint32_t round_count() {
    std::uint32_t r = 0;
    check(lgd_round_count(ctx_, &r));
    return r;
  }
  // one round: this rank's buckets, the next round's NVLink pulls, lock-step relations
  EpochResult train_round(std::uint32_t epoch, std::uint32_t round, double* handoff_ms = nullptr,
                          std::uint64_t* handoff_bytes = nullptr) {
    EpochResult r{};
    check(lgd_train_round(ctx_, epoch, round, &r, handoff_ms, handoff_bytes));
    return r;
  }

  lgd_context* handle() const { return ctx_; }

 private:
  lgd_context* ctx_ = nullptr;
  ScoreModel model_;
};

inline std::vector<unsigned char> comm_unique_id() {
  std::vector<unsigned char> id(128);
  check(lgd_comm_unique_id(id.data()));
  return id;
}

// ingest (graph.cpp:39-118): a TSV edge list on host threads.
struct IngestedGraph {
  std::vector<std::uint32_t> edges;  // 3 per edge: src, rel, dst
  std::uint64_t num_nodes = 0, num_relations = 0;
};
inline IngestedGraph ingest_tsv(const std::string& path, bool triples, bool remap_ids = false,
                                int threads = 0) {
  std::uint32_t* e = nullptr;
  std::uint64_t n = 0;
  IngestedGraph g;
  check(lgd_ingest_tsv(path.c_str(), triples ? 1 : 0, remap_ids ? 1 : 0, threads, &e, &n,
                       &g.num_nodes, &g.num_relations));
  g.edges.assign(e, e + 3 * n);
  lgd_free_edges(e);
  return g;
}
// write_graph / read_graph (graph.cpp:152-192): edges.bin + graph_meta.json.
inline void write_graph(const std::string& dir, const std::vector<std::uint32_t>& edges,
                        std::uint64_t num_nodes, std::uint64_t num_relations) {
  check(lgd_write_graph(dir.c_str(), edges.data(), edges.size() / 3, num_nodes, num_relations));
}
inline IngestedGraph read_graph(const std::string& dir) {
  IngestedGraph g;
  std::uint64_t n = 0;
  check(lgd_read_graph_meta(dir.c_str(), &n, &g.num_nodes, &g.num_relations));
  g.edges.resize(3 * n);
  check(lgd_read_graph(dir.c_str(), g.edges.data(), n));
  return g;
}

// The reference's Algorithms 1-2 (ordering.hpp:49-54) as flat arrays.
struct Plan {
  std::vector<std::uint32_t> states, swaps, bucket_order;
  std::vector<std::uint64_t> state_offsets, prefetch_points;
};
inline Plan plan_iteration_order(std::uint32_t n) {
  std::uint64_t S = 0;
  check(lgd_plan_iteration_order(n, 0, &S, nullptr, nullptr, nullptr, nullptr, nullptr));
  Plan p;
  p.states.resize(3 * S);
  p.swaps.resize(2 * (S ? S - 1 : 0));
  p.bucket_order.resize(2 * std::size_t(n) * n);
  p.state_offsets.resize(S + 1);
  p.prefetch_points.resize(S ? S - 1 : 0);
  check(lgd_plan_iteration_order(n, S, &S, p.states.data(), p.swaps.data(), p.bucket_order.data(),
                                 p.state_offsets.data(), p.prefetch_points.data()));
  return p;
}

}  // namespace legend_b200
