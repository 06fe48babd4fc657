// legend_reference_adapter.cpp -- see legend_reference_adapter.hpp.
#include "legend_reference_adapter.hpp"

#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "legend_b200.h"

namespace legend_b200 {

namespace {

// LGD_* codes -> the reference's exception classes
void check(int rc) {
  if (rc == LGD_OK) return;
  const std::string msg = lgd_last_error();
  switch (rc) {
    case LGD_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case LGD_LOGIC_ERROR: throw std::logic_error(msg);
    case LGD_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

struct Context {
  lgd_context* ctx = nullptr;
  ~Context() { lgd_destroy(ctx); }
};

int kind_of(const legend::ScoreModel& m) {
  switch (m.kind) {
    case legend::ScoreKind::kDot: return LGD_MODEL_DOT;
    case legend::ScoreKind::kDistMult: return LGD_MODEL_DISTMULT;
    default: return LGD_MODEL_COMPLEX;
  }
}

// the store's E||S partitions and relations into the device tables
void upload_store(lgd_context* ctx, const legend::EmbeddingStore& store) {
  for (legend::PartitionId p = 0; p < store.n(); ++p) {
    const legend::EmbeddingPartition part = store.load_partition(p);
    std::vector<float> blob(part.embeddings);
    blob.insert(blob.end(), part.opt_states.begin(), part.opt_states.end());
    check(lgd_load_partition(ctx, p, blob.data(), part.node_count));
  }
  if (store.num_relations()) {
    const legend::RelationTable rt = store.load_relations();
    std::vector<float> blob(rt.embeddings);
    blob.insert(blob.end(), rt.opt_states.begin(), rt.opt_states.end());
    check(lgd_set_relations(ctx, blob.data(), rt.count));
  }
}

std::vector<uint32_t> edge_words(std::span<const legend::Edge> edges) {
  std::vector<uint32_t> e(3 * edges.size());
  for (size_t i = 0; i < edges.size(); ++i) {
    e[3 * i] = edges[i].src;
    e[3 * i + 1] = edges[i].rel;
    e[3 * i + 2] = edges[i].dst;
  }
  return e;
}

}  // namespace

legend::EpochResult run_epoch(const legend::IterationPlan& plan, legend::EmbeddingStore& store,
                              const legend::Graph& graph, const legend::PartitionPlan& parts,
                              const legend::ScoreModel& model, const legend::CostModel& cost,
                              legend::EpochMode mode, const legend::TrainOptions& train,
                              bool prefetch, int device) {
  if (mode == legend::EpochMode::kCostOnly)  // modeled time only: the reference's simulator
    return legend::run_epoch(plan, store, graph, parts, model, cost, mode, train, prefetch);
  const auto t0 = std::chrono::steady_clock::now();
  model.validate();
  if (parts.n != store.n()) throw std::invalid_argument("partition count mismatch");
  if (model.dim != store.dim()) throw std::invalid_argument("dimension mismatch");
  const lgd_train_options o{train.learning_rate, train.adagrad_epsilon, train.batch_size,
                            train.negatives, train.shuffle ? 1 : 0, 0, train.seed};
  Context c;
  check(lgd_create(&c.ctx, kind_of(model), model.dim, &o, device));
  const std::vector<uint32_t> e = edge_words(graph.edges);
  check(lgd_set_graph(c.ctx, e.data(), graph.edges.size(), graph.num_nodes, graph.num_relations));
  check(lgd_set_partition_plan(c.ctx, parts.n, parts.bucket_offsets.data(), parts.edge_order.data()));
  // the caller's IterationPlan, as is
  const auto& seq = plan.buffer_seq;
  std::vector<uint32_t> states, swaps, order;
  for (const auto& s : seq.states) states.insert(states.end(), s.begin(), s.end());
  for (const auto& w : seq.swaps) {
    swaps.push_back(w.evicted);
    swaps.push_back(w.loaded);
  }
  for (const auto& [i, j] : plan.bucket_order) {
    order.push_back(i);
    order.push_back(j);
  }
  check(lgd_set_iteration_plan(c.ctx, seq.states.size(), states.data(),
                               swaps.empty() ? nullptr : swaps.data(), order.data(),
                               plan.state_offsets.data(),
                               plan.prefetch_points.empty() ? nullptr : plan.prefetch_points.data()));
  upload_store(c.ctx, store);
  lgd_epoch_result r{};
  check(lgd_train_epoch(c.ctx, train.epoch, &r));
  // drain: every partition and the relations back to the store (pipeline.cpp:316-322)
  for (legend::PartitionId p = 0; p < store.n(); ++p) {
    legend::EmbeddingPartition part;
    part.id = p;
    part.dim = model.dim;
    part.node_count = store.part_node_count(p);
    std::vector<float> blob(2 * part.node_count * model.dim);
    check(lgd_store_partition(c.ctx, p, blob.data(), part.node_count));
    const size_t half = part.node_count * model.dim;
    part.embeddings.assign(blob.begin(), blob.begin() + half);
    part.opt_states.assign(blob.begin() + half, blob.end());
    store.save_partition(part);
  }
  if (store.num_relations()) {
    legend::RelationTable rt = store.load_relations();
    std::vector<float> blob(2 * rt.count * model.dim);
    check(lgd_get_relations(c.ctx, blob.data(), rt.count));
    const size_t half = rt.count * model.dim;
    rt.embeddings.assign(blob.begin(), blob.begin() + half);
    rt.opt_states.assign(blob.begin() + half, blob.end());
    store.save_relations(rt);
  }
  legend::EpochResult out;
  out.loss_sum = r.loss_sum;
  out.loss_per_edge = r.loss_per_edge;
  out.edges_trained = r.edges_trained;
  out.buckets_trained = r.buckets_trained;
  out.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return out;
}

legend::EvalResult evaluate(const legend::ScoreModel& model, const legend::EmbeddingStore& store,
                            std::span<const legend::Edge> test_edges,
                            const legend::EvalOptions& options, int device) {
  model.validate();
  if (test_edges.empty()) throw std::invalid_argument("test edge set is empty");
  if (options.num_candidates == 0) throw std::invalid_argument("need at least one candidate");
  const lgd_train_options o{0.1, 1e-10, 100000, 16, 1, 0, 0};
  Context c;
  check(lgd_create(&c.ctx, kind_of(model), model.dim, &o, device));
  // the store's node count and partitioning, no edges: an empty graph
  const uint32_t none[3] = {0, 0, 0};
  check(lgd_set_graph(c.ctx, none, 0, store.num_nodes(), store.num_relations()));
  std::vector<uint64_t> offsets(uint64_t(store.n()) * store.n() + 1, 0);
  check(lgd_set_partition_plan(c.ctx, store.n(), offsets.data(), offsets.data()));
  upload_store(c.ctx, store);
  const std::vector<uint32_t> e = edge_words(test_edges);
  legend::EvalResult r;
  r.edges = test_edges.size();
  check(lgd_evaluate(c.ctx, e.data(), test_edges.size(), options.num_candidates, options.hits_k,
                     options.seed, &r.mrr, &r.hits_at_k));
  return r;
}

}  // namespace legend_b200
