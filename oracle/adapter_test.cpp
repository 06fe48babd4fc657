// adapter_test.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The reference's drop-in check for run_epoch ("out-of-core epoch equals the
// in-memory reference", proj/tests/test_pipeline.cpp:197-289), restated with
// the B200 adapter (adapters/legend_reference_adapter.hpp) in place of
// legend::run_epoch: same reference types, same plan / store / graph objects.
// The in-memory restatement is driven by the UNMODIFIED reference primitives
// (sample_negatives / batch_loss / batch_gradients / adagrad_step from
// oracle/_ref/liblegend_ref.so).  Also checks legend_b200::evaluate against
// legend::evaluate on the trained store.  Built by oracle/Makefile (target
// adapter) where the reference sources exist; run on the GPU box by
// tests/test_gpu_adapter.py.
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <string>
#include <vector>

#include "../adapters/legend_reference_adapter.hpp"
#include "legend/rng.hpp"

using namespace legend;
namespace fs = std::filesystem;

static int failures = 0;
#define EXPECT(cond, ...)                                    \
  do {                                                       \
    if (!(cond)) {                                           \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__);       \
      std::printf(__VA_ARGS__);                              \
      std::printf("\n");                                     \
      ++failures;                                            \
    }                                                        \
  } while (0)

static Graph random_graph(std::uint64_t nodes, std::uint64_t edges, std::uint32_t rels,
                          std::uint64_t seed) {
  Graph g;
  g.num_nodes = nodes;
  g.num_relations = rels;
  Rng rng(seed);
  for (std::uint64_t i = 0; i < edges; ++i) {
    const NodeId s = static_cast<NodeId>(rng.next_below(nodes));
    const RelId r = rels ? static_cast<RelId>(rng.next_below(rels)) : kNoRelation;
    // a few hubs so some rows collect many contributions per batch
    const NodeId t = rng.next_below(4) == 0 ? static_cast<NodeId>(rng.next_below(8))
                                            : static_cast<NodeId>(rng.next_below(nodes));
    g.edges.push_back({s, r, t});
  }
  return g;
}

static void check_model(ScoreKind kind, std::uint32_t dim, std::uint32_t n, const fs::path& dir) {
  const char* name = score_kind_name(kind);
  const std::uint32_t rels = kind == ScoreKind::kDot ? 0 : 6;
  const Graph g = random_graph(600, 8000, rels, 11);
  const PartitionPlan parts = make_partition_plan(g, n);
  const ScoreModel model{kind, dim};
  const IterationPlan plan = plan_iteration_order(plan_loading_order(n), n);
  EmbeddingStore store =
      EmbeddingStore::create(parts, dim, g.num_relations, 77, dir / (std::string(name) + "_gpu"));
  EmbeddingStore mirror =
      EmbeddingStore::create(parts, dim, g.num_relations, 77, dir / (std::string(name) + "_ref"));
  TrainOptions opts;
  opts.learning_rate = 0.1;
  opts.batch_size = 300;
  opts.negatives = 5;
  opts.shuffle = true;
  opts.seed = 5;
  opts.epoch = 0;
  CostModel cost;
  cost.dim = dim;

  const EpochResult res =
      legend_b200::run_epoch(plan, store, g, parts, model, cost, EpochMode::kRealTrain, opts);
  EXPECT(res.edges_trained == g.edges.size(), "%s edges %llu", name,
         (unsigned long long)res.edges_trained);

  // the in-memory restatement (test_pipeline.cpp:227-269) on the reference primitives
  ResidentTable full(dim);
  for (PartitionId p = 0; p < n; ++p) full.add_partition(mirror.load_partition(p), mirror.part_begin(p));
  if (rels) full.set_relations(mirror.load_relations());
  const AdagradHyper hyper{opts.learning_rate, opts.adagrad_epsilon};
  const auto& seq = plan.buffer_seq;
  std::size_t state = 0;
  double ref_loss = 0.0;
  std::uint64_t buckets = 0;
  for (std::size_t gi = 0; gi < plan.bucket_order.size(); ++gi) {
    while (state + 1 < seq.states.size() && gi >= plan.state_offsets[state + 1]) ++state;
    ResidentTable skeleton(dim);
    for (PartitionId p : seq.states[state]) {
      EmbeddingPartition stub;
      stub.id = p;
      stub.dim = dim;
      stub.node_count = parts.part_node_count(p);
      stub.embeddings.assign(stub.node_count * dim, 0.0f);
      stub.opt_states.assign(stub.node_count * dim, 0.0f);
      skeleton.add_partition(std::move(stub), parts.part_begin(p));
    }
    const auto [bi, bj] = plan.bucket_order[gi];
    const auto ids = parts.bucket(bi, bj);
    if (ids.empty()) continue;
    ++buckets;
    std::vector<Edge> edges;
    for (std::uint64_t idx : ids) edges.push_back(g.edges[idx]);
    Rng rng(derive_seed(opts.seed, 0x62756b74ull, opts.epoch, gi));
    for (std::size_t i = edges.size(); i > 1; --i) std::swap(edges[i - 1], edges[rng.next_below(i)]);
    for (std::size_t off = 0; off < edges.size(); off += opts.batch_size) {
      const std::size_t count = std::min<std::size_t>(opts.batch_size, edges.size() - off);
      TrainBatch batch;
      batch.positives.assign(edges.begin() + off, edges.begin() + off + count);
      batch.negatives_per_positive = opts.negatives;
      batch.negative_dst = sample_negatives(skeleton, opts.negatives, count, rng);
      ref_loss += batch_loss(model, batch, full);
      adagrad_step(full, batch_gradients(model, batch, full), hyper);
    }
  }
  EXPECT(res.buckets_trained == buckets, "%s buckets", name);
  const double lrel = std::fabs(res.loss_sum - ref_loss) / std::fabs(ref_loss);
  EXPECT(lrel <= 1e-12, "%s loss %.17g vs %.17g (rel %.3g)", name, res.loss_sum, ref_loss, lrel);

  // every row of every partition: bit-identical, or within the stated tolerance
  std::uint64_t same = 0, total = 0;
  double num = 0.0, den = 0.0;
  for (PartitionId p = 0; p < n; ++p) {
    const EmbeddingPartition trained = store.load_partition(p);
    for (std::uint64_t v = parts.part_begin(p); v < parts.part_end(p); ++v) {
      const auto want = full.node_embedding(static_cast<NodeId>(v));
      const float* got = trained.embeddings.data() + (v - parts.part_begin(p)) * dim;
      for (std::uint32_t i = 0; i < dim; ++i) {
        same += std::memcmp(got + i, want.data() + i, 4) == 0;
        ++total;
        num += (double(got[i]) - want[i]) * (double(got[i]) - want[i]);
        den += double(want[i]) * want[i];
      }
    }
  }
  const double frob = std::sqrt(num / den);
  EXPECT(frob <= 1e-7 && same >= 0.99 * total, "%s rows: frob %.3g, %llu/%llu identical", name,
         frob, (unsigned long long)same, (unsigned long long)total);

  // evaluate on the trained store: the adapter against the reference
  std::vector<Edge> test(g.edges.begin(), g.edges.begin() + 400);
  EvalOptions eo;
  eo.num_candidates = 199;
  eo.hits_k = 10;
  eo.seed = 3;
  const EvalResult eg = legend_b200::evaluate(model, store, test, eo);
  const EvalResult er = legend::evaluate(model, store, test, eo);
  EXPECT(eg.mrr == er.mrr && eg.hits_at_k == er.hits_at_k && eg.edges == er.edges,
         "%s evaluate %.17g/%.17g vs %.17g/%.17g", name, eg.mrr, eg.hits_at_k, er.mrr,
         er.hits_at_k);
  std::printf("adapter %s: loss rel %.2g, rows %llu/%llu bit-identical (frob %.2g), MRR %.6f == %.6f\n",
              name, lrel, (unsigned long long)same, (unsigned long long)total, frob, eg.mrr, er.mrr);
}

int main() {
  const fs::path dir = fs::temp_directory_path() / ("lgd_adapter_" + std::to_string(::getpid()));
  fs::create_directories(dir);
  try {
    check_model(ScoreKind::kDistMult, 12, 4, dir);
    check_model(ScoreKind::kComplEx, 12, 5, dir);
    check_model(ScoreKind::kDot, 8, 6, dir);
  } catch (const std::exception& e) {
    std::printf("FAIL exception: %s\n", e.what());
    ++failures;
  }
  fs::remove_all(dir);
  std::printf(failures ? "adapter FAILED (%d)\n" : "adapter ok\n", failures);
  return failures ? 1 : 0;
}
