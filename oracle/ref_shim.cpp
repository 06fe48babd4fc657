// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/liblegend_ref.so).  Python (ctypes) uses it to generate the
// golden vectors in tests/golden/ and to pin the C restatement in
// oracle/legend_oracle.c.  Every entry point forwards to the reference API
// named in its comment; nothing here re-implements reference arithmetic,
// except ref_run_epoch_inmem, which is the reference test suite's own
// all-resident restatement of run_epoch (test_pipeline.cpp:227-269) driven
// through the reference primitives.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "legend/graph.hpp"
#include "legend/ordering.hpp"
#include "legend/pipeline.hpp"
#include "legend/rng.hpp"
#include "legend/store.hpp"
#include "legend/train.hpp"

using namespace legend;
namespace fs = std::filesystem;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

ScoreModel model_of(int kind, std::uint32_t dim) {
  ScoreModel m;
  m.kind = kind == 0 ? ScoreKind::kDot : (kind == 1 ? ScoreKind::kDistMult : ScoreKind::kComplEx);
  m.dim = dim;
  return m;
}

std::vector<Edge> edges_of(const std::uint32_t* e, std::uint64_t count) {
  std::vector<Edge> out(count);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = {e[3 * i], e[3 * i + 1], e[3 * i + 2]};
  return out;
}

ResidentTable table_of(std::uint32_t dim, const float* E, const float* S, std::uint64_t nodes,
                       const float* relE, const float* relS, std::uint64_t rels) {
  ResidentTable t(dim);
  EmbeddingPartition part;
  part.id = 0;
  part.dim = dim;
  part.node_count = nodes;
  part.embeddings.assign(E, E + nodes * dim);
  part.opt_states.assign(S, S + nodes * dim);
  t.add_partition(std::move(part), 0);
  RelationTable rt;
  rt.dim = dim;
  rt.count = rels;
  if (rels) {
    rt.embeddings.assign(relE, relE + rels * dim);
    rt.opt_states.assign(relS, relS + rels * dim);
  }
  t.set_relations(std::move(rt));
  return t;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// rng.hpp:57-67
std::uint64_t ref_derive_seed(std::uint64_t base, std::uint64_t a, std::uint64_t b,
                              std::uint64_t c) {
  return derive_seed(base, a, b, c);
}

// rng.hpp:23-33
void ref_rng_u64(std::uint64_t seed, std::uint64_t skip, std::uint64_t n, std::uint64_t* out) {
  Rng r(seed);
  for (std::uint64_t i = 0; i < skip; ++i) r.next_u64();
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

// rng.hpp:42-48 (consumed is inferred by replaying the raw stream)
void ref_rng_below_seq(std::uint64_t seed, std::uint64_t skip, const std::uint64_t* bounds,
                       std::uint64_t n, std::uint64_t* out, std::uint64_t* consumed) {
  Rng r(seed);
  for (std::uint64_t i = 0; i < skip; ++i) r.next_u64();
  for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next_below(bounds[i]);
  if (consumed) {
    // count raw draws: advance a twin stream until it matches r's next output
    Rng twin(seed);
    for (std::uint64_t i = 0; i < skip; ++i) twin.next_u64();
    Rng probe = r;
    const std::uint64_t target = probe.next_u64();
    std::uint64_t used = 0;
    while (twin.next_u64() != target) ++used;
    *consumed = used;
  }
}

// graph.cpp:120-150
int ref_partition_plan(const std::uint32_t* edges, std::uint64_t num_edges,
                       std::uint64_t num_nodes, std::uint32_t n, std::uint64_t* stride,
                       std::uint64_t* offsets, std::uint64_t* edge_order) {
  return guarded([&] {
    Graph g;
    g.num_nodes = num_nodes;
    g.edges = edges_of(edges, num_edges);
    const PartitionPlan plan = make_partition_plan(g, n);
    *stride = plan.stride;
    std::memcpy(offsets, plan.bucket_offsets.data(), plan.bucket_offsets.size() * 8);
    std::memcpy(edge_order, plan.edge_order.data(), plan.edge_order.size() * 8);
  });
}

// store.cpp:59-102 EmbeddingStore::create, then load_partition / load_relations
int ref_store_init(const char* dir, std::uint32_t n, std::uint64_t num_nodes, std::uint32_t dim,
                   std::uint64_t num_relations, std::uint64_t seed, float* E, float* S,
                   float* relE, float* relS) {
  return guarded([&] {
    PartitionPlan plan;
    plan.n = n;
    plan.num_nodes = num_nodes;
    plan.stride = (num_nodes + n - 1) / n;
    EmbeddingStore store = EmbeddingStore::create(plan, dim, num_relations, seed, dir);
    for (PartitionId p = 0; p < n; ++p) {
      const EmbeddingPartition part = store.load_partition(p);
      const std::uint64_t off = store.part_begin(p) * dim;
      std::memcpy(E + off, part.embeddings.data(), part.embeddings.size() * 4);
      std::memcpy(S + off, part.opt_states.data(), part.opt_states.size() * 4);
    }
    if (num_relations) {
      const RelationTable rt = store.load_relations();
      std::memcpy(relE, rt.embeddings.data(), rt.embeddings.size() * 4);
      std::memcpy(relS, rt.opt_states.data(), rt.opt_states.size() * 4);
    }
  });
}

// train.cpp:365-373 over resident ranges (train.cpp:112-119, 190-202)
int ref_sample_negatives(const std::uint64_t* first, const std::uint64_t* count, int nparts,
                         std::uint32_t k, std::uint64_t num_positives, std::uint64_t seed,
                         std::uint64_t skip, std::uint32_t* out) {
  return guarded([&] {
    ResidentTable t(1);
    for (int i = 0; i < nparts; ++i) {
      EmbeddingPartition p;
      p.id = static_cast<PartitionId>(i);
      p.dim = 1;
      p.node_count = count[i];
      p.embeddings.assign(count[i], 0.0f);
      p.opt_states.assign(count[i], 0.0f);
      t.add_partition(std::move(p), first[i]);
    }
    Rng rng(seed);
    for (std::uint64_t i = 0; i < skip; ++i) rng.next_u64();
    const auto ids = sample_negatives(t, k, num_positives, rng);
    std::memcpy(out, ids.data(), ids.size() * 4);
  });
}

// batch_loss (train.cpp:217-278) + batch_gradients (280-340) + adagrad_step (356-363)
int ref_batch(int kind, std::uint32_t d, float* E, float* S, std::uint64_t num_nodes,
              float* relE, float* relS, std::uint64_t num_rels, const std::uint32_t* edges,
              std::uint64_t P, const std::uint32_t* negs, std::uint32_t k, double lr, double eps,
              int apply, double* loss_out, std::uint64_t* n_nodes_out, std::uint32_t* node_ids,
              double* node_grads, std::uint64_t* n_rels_out, std::uint32_t* rel_ids,
              double* rel_grads) {
  return guarded([&] {
    const ScoreModel model = model_of(kind, d);
    ResidentTable table = table_of(d, E, S, num_nodes, relE, relS, num_rels);
    TrainBatch batch;
    batch.positives = edges_of(edges, P);
    batch.negatives_per_positive = k;
    batch.negative_dst.assign(negs, negs + P * k);
    const double loss = batch_loss(model, batch, table);
    const GradientSet gs = batch_gradients(model, batch, table);
    if (loss_out) *loss_out = loss;
    if (n_nodes_out) *n_nodes_out = gs.nodes.size();
    if (n_rels_out) *n_rels_out = gs.rels.size();
    for (std::size_t u = 0; u < gs.nodes.size(); ++u) {
      if (node_ids) node_ids[u] = gs.nodes[u].first;
      if (node_grads) std::memcpy(node_grads + u * d, gs.nodes[u].second.data(), d * 8);
    }
    for (std::size_t u = 0; u < gs.rels.size(); ++u) {
      if (rel_ids) rel_ids[u] = gs.rels[u].first;
      if (rel_grads) std::memcpy(rel_grads + u * d, gs.rels[u].second.data(), d * 8);
    }
    if (apply) {
      adagrad_step(table, gs, AdagradHyper{lr, eps});
      const auto e0 = table.node_embedding(0);
      const auto s0 = table.node_acc(0);
      std::memcpy(E, e0.data(), num_nodes * d * 4);
      std::memcpy(S, s0.data(), num_nodes * d * 4);
      if (num_rels) {
        std::memcpy(relE, table.relations().embeddings.data(), num_rels * d * 4);
        std::memcpy(relS, table.relations().opt_states.data(), num_rels * d * 4);
      }
    }
  });
}

// plan_loading_order (ordering.cpp:59-156) + plan_iteration_order (245-346).
// Call with cap == 0 to learn num_states.
int ref_iteration_plan(std::uint32_t n, std::uint64_t cap, std::uint64_t* num_states,
                       std::uint32_t* states, std::uint32_t* swaps, std::uint32_t* bucket_order,
                       std::uint64_t* state_offsets, std::uint64_t* prefetch_points) {
  return guarded([&] {
    const IterationPlan plan = plan_iteration_order(plan_loading_order(n), n);
    const std::uint64_t S = plan.buffer_seq.states.size();
    *num_states = S;
    if (cap < S) return;
    for (std::uint64_t i = 0; i < S; ++i)
      for (int j = 0; j < 3; ++j) states[3 * i + j] = plan.buffer_seq.states[i][j];
    for (std::uint64_t i = 0; i + 1 < S; ++i) {
      swaps[2 * i] = plan.buffer_seq.swaps[i].evicted;
      swaps[2 * i + 1] = plan.buffer_seq.swaps[i].loaded;
    }
    for (std::size_t g = 0; g < plan.bucket_order.size(); ++g) {
      bucket_order[2 * g] = plan.bucket_order[g].first;
      bucket_order[2 * g + 1] = plan.bucket_order[g].second;
    }
    std::memcpy(state_offsets, plan.state_offsets.data(), (S + 1) * 8);
    std::memcpy(prefetch_points, plan.prefetch_points.data(), (S - 1) * 8);
  });
}

// plan_to_json (ordering.cpp:428-440)
int ref_plan_json(std::uint32_t n, char* buf, std::uint64_t cap, std::uint64_t* len) {
  return guarded([&] {
    const std::string s = plan_to_json(plan_iteration_order(plan_loading_order(n), n));
    *len = s.size();
    if (cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

// verify_prefetchable (ordering.cpp:348-418): returns report.ok
int ref_verify_prefetchable(std::uint32_t n, std::uint64_t num_states, const std::uint32_t* states,
                            const std::uint32_t* swaps, const std::uint32_t* bucket_order,
                            const std::uint64_t* state_offsets,
                            const std::uint64_t* prefetch_points, int* ok) {
  return guarded([&] {
    IterationPlan plan;
    plan.buffer_seq.n = n;
    for (std::uint64_t i = 0; i < num_states; ++i)
      plan.buffer_seq.states.push_back({states[3 * i], states[3 * i + 1], states[3 * i + 2]});
    for (std::uint64_t i = 0; i + 1 < num_states; ++i)
      plan.buffer_seq.swaps.push_back({swaps[2 * i], swaps[2 * i + 1]});
    for (std::uint64_t g = 0; g < std::uint64_t(n) * n; ++g)
      plan.bucket_order.push_back({bucket_order[2 * g], bucket_order[2 * g + 1]});
    plan.state_offsets.assign(state_offsets, state_offsets + num_states + 1);
    plan.prefetch_points.assign(prefetch_points, prefetch_points + num_states - 1);
    *ok = verify_prefetchable(plan).ok ? 1 : 0;
  });
}

// run_epoch real-train (pipeline.cpp:215-333) through a real on-disk store
// under dir: EmbeddingStore::create(seed), one epoch, then the trained E||S
// read back.  Requires n >= 4 (plan_loading_order).
int ref_run_epoch_store(const char* dir, const std::uint32_t* edges, std::uint64_t num_edges,
                        std::uint64_t num_nodes, std::uint64_t num_rels, std::uint32_t n,
                        int kind, std::uint32_t d, double lr, double eps,
                        std::uint32_t batch_size, std::uint32_t k, int shuffle,
                        std::uint64_t train_seed, std::uint32_t epoch, std::uint64_t store_seed,
                        float* E, float* S, float* relE, float* relS, double* loss_sum,
                        std::uint64_t* edges_trained, std::uint64_t* buckets_trained) {
  return guarded([&] {
    Graph g;
    g.num_nodes = num_nodes;
    g.num_relations = num_rels;
    g.edges = edges_of(edges, num_edges);
    const PartitionPlan parts = make_partition_plan(g, n);
    const ScoreModel model = model_of(kind, d);
    const IterationPlan plan = plan_iteration_order(plan_loading_order(n), n);
    EmbeddingStore store = EmbeddingStore::create(parts, d, num_rels, store_seed, dir);
    TrainOptions opts;
    opts.learning_rate = lr;
    opts.adagrad_epsilon = eps;
    opts.batch_size = batch_size;
    opts.negatives = k;
    opts.shuffle = shuffle != 0;
    opts.seed = train_seed;
    opts.epoch = epoch;
    CostModel cost;
    cost.dim = d;
    const EpochResult res =
        run_epoch(plan, store, g, parts, model, cost, EpochMode::kRealTrain, opts);
    *loss_sum = res.loss_sum;
    *edges_trained = res.edges_trained;
    *buckets_trained = res.buckets_trained;
    for (PartitionId p = 0; p < n; ++p) {
      const EmbeddingPartition part = store.load_partition(p);
      const std::uint64_t off = store.part_begin(p) * d;
      std::memcpy(E + off, part.embeddings.data(), part.embeddings.size() * 4);
      std::memcpy(S + off, part.opt_states.data(), part.opt_states.size() * 4);
    }
    if (num_rels) {
      const RelationTable rt = store.load_relations();
      std::memcpy(relE, rt.embeddings.data(), rt.embeddings.size() * 4);
      std::memcpy(relS, rt.opt_states.data(), rt.opt_states.size() * 4);
    }
  });
}

// The reference suite's all-resident epoch restatement (test_pipeline.cpp:
// 227-269) generalised to any plan (states may list fewer than 3 partitions,
// 0xffffffff = empty slot, so n <= 3 runs as a single all-resident state).
// Drives the reference's own Rng, sample_negatives, batch_loss,
// batch_gradients and adagrad_step; dumps per-batch losses, unique-row
// counts, in-bucket shuffled positions and negative ids for the golden files.
int ref_run_epoch_inmem(const std::uint32_t* edges, std::uint64_t num_edges,
                        std::uint64_t num_nodes, std::uint64_t num_rels, std::uint32_t n,
                        std::uint64_t num_states, const std::uint32_t* states,
                        const std::uint32_t* bucket_order, const std::uint64_t* state_offsets,
                        int kind, std::uint32_t d, double lr, double eps,
                        std::uint32_t batch_size, std::uint32_t k, int shuffle,
                        std::uint64_t seed, std::uint32_t epoch, float* E, float* S,
                        float* relE, float* relS, double* loss_sum_out,
                        std::uint64_t* edges_trained_out, std::uint64_t* buckets_trained_out,
                        std::uint64_t* num_batches_out, std::uint64_t max_batches,
                        double* batch_loss_out, std::uint64_t* batch_nodes,
                        std::uint64_t* batch_rels, std::uint32_t* perm_dump,
                        std::uint32_t* neg_dump) {
  return guarded([&] {
    Graph g;
    g.num_nodes = num_nodes;
    g.num_relations = num_rels;
    g.edges = edges_of(edges, num_edges);
    const PartitionPlan parts = make_partition_plan(g, n);
    const ScoreModel model = model_of(kind, d);
    if (model.uses_relations() && num_rels == 0)
      throw std::invalid_argument("typed model on a store without relation embeddings");
    ResidentTable full = table_of(d, E, S, num_nodes, relE, relS, num_rels);
    const AdagradHyper hyper{lr, eps};
    std::size_t state = 0;
    double loss_sum = 0.0;
    std::uint64_t edges_trained = 0, buckets_trained = 0, nb = 0, perm_pos = 0, neg_pos = 0;
    for (std::size_t gidx = 0; gidx < std::size_t(n) * n; ++gidx) {
      while (state + 1 < num_states && gidx >= state_offsets[state + 1]) ++state;
      ResidentTable skeleton(d);
      for (int s2 = 0; s2 < 3; ++s2) {
        const std::uint32_t p = states[3 * state + s2];
        if (p == 0xffffffffu) continue;
        EmbeddingPartition stub;
        stub.id = p;
        stub.dim = d;
        stub.node_count = parts.part_node_count(p);
        stub.embeddings.assign(stub.node_count * d, 0.0f);
        stub.opt_states.assign(stub.node_count * d, 0.0f);
        skeleton.add_partition(std::move(stub), parts.part_begin(p));
      }
      const PartitionId bi = bucket_order[2 * gidx], bj = bucket_order[2 * gidx + 1];
      const auto ids = parts.bucket(bi, bj);
      if (ids.empty()) continue;
      std::vector<Edge> bucket;
      std::vector<std::uint32_t> pos(ids.size());
      for (std::size_t i = 0; i < ids.size(); ++i) {
        bucket.push_back(g.edges[ids[i]]);
        pos[i] = static_cast<std::uint32_t>(i);
      }
      Rng rng(derive_seed(seed, 0x62756b74ull, epoch, gidx));
      if (shuffle) {
        for (std::size_t i = bucket.size(); i > 1; --i) {
          const std::uint64_t j = rng.next_below(i);
          std::swap(bucket[i - 1], bucket[j]);
          std::swap(pos[i - 1], pos[j]);
        }
      }
      if (perm_dump) std::memcpy(perm_dump + perm_pos, pos.data(), pos.size() * 4);
      perm_pos += pos.size();
      for (std::size_t off = 0; off < bucket.size(); off += batch_size) {
        const std::size_t count = std::min<std::size_t>(batch_size, bucket.size() - off);
        TrainBatch batch;
        batch.positives.assign(bucket.begin() + off, bucket.begin() + off + count);
        batch.negatives_per_positive = k;
        batch.negative_dst = sample_negatives(skeleton, k, count, rng);
        if (neg_dump)
          std::memcpy(neg_dump + neg_pos, batch.negative_dst.data(),
                      batch.negative_dst.size() * 4);
        neg_pos += batch.negative_dst.size();
        const double l = batch_loss(model, batch, full);
        const GradientSet gs = batch_gradients(model, batch, full);
        adagrad_step(full, gs, hyper);
        if (nb < max_batches) {
          if (batch_loss_out) batch_loss_out[nb] = l;
          if (batch_nodes) batch_nodes[nb] = gs.nodes.size();
          if (batch_rels) batch_rels[nb] = gs.rels.size();
        }
        ++nb;
        loss_sum += l;
      }
      edges_trained += bucket.size();
      ++buckets_trained;
    }
    *loss_sum_out = loss_sum;
    *edges_trained_out = edges_trained;
    *buckets_trained_out = buckets_trained;
    *num_batches_out = nb;
    std::memcpy(E, full.node_embedding(0).data(), num_nodes * d * 4);
    std::memcpy(S, full.node_acc(0).data(), num_nodes * d * 4);
    if (num_rels) {
      std::memcpy(relE, full.relations().embeddings.data(), num_rels * d * 4);
      std::memcpy(relS, full.relations().opt_states.data(), num_rels * d * 4);
    }
  });
}

// Bounded CPU-baseline sample through the reference primitives: one bucket's
// copy + shuffle (pipeline.cpp:293-301) and up to max_batches batches of
// sample_negatives + batch_loss + batch_gradients + adagrad_step
// (pipeline.cpp:303-312).  The table holds rows [0, num_nodes).
int ref_bucket_sample(const std::uint32_t* bucket_edges, std::uint64_t m,
                      const std::uint64_t* first, const std::uint64_t* count, int nparts,
                      std::uint64_t stream_seed, int shuffle, std::uint32_t batch_size,
                      std::uint32_t k, std::uint64_t max_batches, int kind, std::uint32_t d,
                      float* E, float* S, std::uint64_t num_nodes, float* relE, float* relS,
                      std::uint64_t num_rels, double lr, double eps, double* loss_sum,
                      std::uint64_t* edges_trained) {
  return guarded([&] {
    const ScoreModel model = model_of(kind, d);
    ResidentTable table = table_of(d, E, S, num_nodes, relE, relS, num_rels);
    ResidentTable pool(1);
    for (int i = 0; i < nparts; ++i) {
      EmbeddingPartition p;
      p.id = static_cast<PartitionId>(i);
      p.dim = 1;
      p.node_count = count[i];
      p.embeddings.assign(count[i], 0.0f);
      p.opt_states.assign(count[i], 0.0f);
      pool.add_partition(std::move(p), first[i]);
    }
    std::vector<Edge> edges = edges_of(bucket_edges, m);
    Rng rng(stream_seed);
    if (shuffle)
      for (std::size_t i = edges.size(); i > 1; --i) std::swap(edges[i - 1], edges[rng.next_below(i)]);
    const AdagradHyper hyper{lr, eps};
    double total = 0.0;
    std::uint64_t done = 0, nb = 0;
    for (std::size_t off = 0; off < edges.size() && nb < max_batches; off += batch_size, ++nb) {
      const std::size_t cnt = std::min<std::size_t>(batch_size, edges.size() - off);
      TrainBatch batch;
      batch.positives.assign(edges.begin() + off, edges.begin() + off + cnt);
      batch.negatives_per_positive = k;
      batch.negative_dst = sample_negatives(pool, k, cnt, rng);
      total += batch_loss(model, batch, table);
      adagrad_step(table, batch_gradients(model, batch, table), hyper);
      done += cnt;
    }
    *loss_sum = total;
    *edges_trained = done;
  });
}

// The same bounded bucket sample with per-batch outputs: the loss of every
// batch (batch_loss) and its wall time in ns around sample_negatives +
// batch_loss + batch_gradients + adagrad_step (the reference arm of bench.py
// times these).  Arrays hold max_batches entries (or fewer when the bucket
// ends first, or once budget_ns > 0 of batch time is spent); the table copy-in
// above the loop is not timed.
int ref_bucket_sample_timed(const std::uint32_t* bucket_edges, std::uint64_t m,
                            const std::uint64_t* first, const std::uint64_t* count, int nparts,
                            std::uint64_t stream_seed, int shuffle, std::uint32_t batch_size,
                            std::uint32_t k, std::uint64_t max_batches, int kind, std::uint32_t d,
                            float* E, float* S, std::uint64_t num_nodes, float* relE, float* relS,
                            std::uint64_t num_rels, double lr, double eps, double* batch_losses,
                            std::uint64_t* batch_ns, std::uint64_t* batches_done,
                            std::uint64_t budget_ns) {
  return guarded([&] {
    const ScoreModel model = model_of(kind, d);
    ResidentTable table = table_of(d, E, S, num_nodes, relE, relS, num_rels);
    ResidentTable pool(1);
    for (int i = 0; i < nparts; ++i) {
      EmbeddingPartition p;
      p.id = static_cast<PartitionId>(i);
      p.dim = 1;
      p.node_count = count[i];
      p.embeddings.assign(count[i], 0.0f);
      p.opt_states.assign(count[i], 0.0f);
      pool.add_partition(std::move(p), first[i]);
    }
    std::vector<Edge> edges = edges_of(bucket_edges, m);
    Rng rng(stream_seed);
    if (shuffle)
      for (std::size_t i = edges.size(); i > 1; --i) std::swap(edges[i - 1], edges[rng.next_below(i)]);
    const AdagradHyper hyper{lr, eps};
    std::uint64_t nb = 0, spent = 0;
    for (std::size_t off = 0; off < edges.size() && nb < max_batches && (!budget_ns || spent < budget_ns);
         off += batch_size, ++nb) {
      const std::size_t cnt = std::min<std::size_t>(batch_size, edges.size() - off);
      const auto t0 = std::chrono::steady_clock::now();
      TrainBatch batch;
      batch.positives.assign(edges.begin() + off, edges.begin() + off + cnt);
      batch.negatives_per_positive = k;
      batch.negative_dst = sample_negatives(pool, k, cnt, rng);
      batch_losses[nb] = batch_loss(model, batch, table);
      adagrad_step(table, batch_gradients(model, batch, table), hyper);
      batch_ns[nb] = (std::uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
                         std::chrono::steady_clock::now() - t0)
                         .count();
      spent += batch_ns[nb];
    }
    *batches_done = nb;
  });
}

// ingest (graph.cpp:39-118) through the reference itself; edges_out holds up
// to cap records
int ref_ingest(const char* path, int triples, int remap, std::uint32_t* edges_out,
               std::uint64_t cap, std::uint64_t* num_edges, std::uint64_t* num_nodes,
               std::uint64_t* num_relations) {
  return guarded([&] {
    IngestOptions o;
    o.remap_ids = remap != 0;
    const Graph g = ingest(path, triples ? EdgeFileFormat::kTriples : EdgeFileFormat::kPairs, o);
    *num_edges = g.edges.size();
    *num_nodes = g.num_nodes;
    *num_relations = g.num_relations;
    for (std::uint64_t i = 0; i < g.edges.size() && i < cap; ++i) {
      edges_out[3 * i] = g.edges[i].src;
      edges_out[3 * i + 1] = g.edges[i].rel;
      edges_out[3 * i + 2] = g.edges[i].dst;
    }
  });
}

// write_graph / read_graph (graph.cpp:152-192) through the reference itself
int ref_write_graph(const char* dir, const std::uint32_t* edges, std::uint64_t num_edges,
                    std::uint64_t num_nodes, std::uint64_t num_relations) {
  return guarded([&] {
    Graph g;
    g.num_nodes = num_nodes;
    g.num_relations = num_relations;
    g.edges = edges_of(edges, num_edges);
    write_graph(g, dir);
  });
}

int ref_read_graph(const char* dir, std::uint32_t* edges_out, std::uint64_t cap,
                   std::uint64_t* num_edges, std::uint64_t* num_nodes,
                   std::uint64_t* num_relations) {
  return guarded([&] {
    const Graph g = read_graph(dir);
    *num_edges = g.edges.size();
    *num_nodes = g.num_nodes;
    *num_relations = g.num_relations;
    for (std::uint64_t i = 0; i < g.edges.size() && i < cap; ++i) {
      edges_out[3 * i] = g.edges[i].src;
      edges_out[3 * i + 1] = g.edges[i].rel;
      edges_out[3 * i + 2] = g.edges[i].dst;
    }
  });
}

// evaluate (train.cpp:375-412) over an all-resident table
int ref_evaluate(int kind, std::uint32_t d, const float* E, std::uint64_t num_nodes,
                 const float* relE, std::uint64_t num_rels, const std::uint32_t* test_edges,
                 std::uint64_t T, std::uint32_t num_candidates, std::uint32_t hits_k,
                 std::uint64_t seed, double* mrr, double* hits) {
  return guarded([&] {
    std::vector<float> zn(num_nodes * d, 0.0f), zr(num_rels * d, 0.0f);
    ResidentTable table = table_of(d, E, zn.data(), num_nodes, relE, zr.data(), num_rels);
    const auto edges = edges_of(test_edges, T);
    EvalOptions opts;
    opts.num_candidates = num_candidates;
    opts.hits_k = hits_k;
    opts.seed = seed;
    const EvalResult r = evaluate(model_of(kind, d), table, edges, opts);
    *mrr = r.mrr;
    *hits = r.hits_at_k;
  });
}

}  // extern "C"
