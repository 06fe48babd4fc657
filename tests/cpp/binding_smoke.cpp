// Compiled and run by tests/test_cpp_binding.py: the C++ face of the C ABI.
// Without a GPU it must throw std::runtime_error (no CPU fallback) after the
// host-only planner works; with a GPU it trains one tiny epoch.
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "legend_b200.hpp"

int main(int argc, char** argv) {
  const bool expect_gpu = argc > 1 && argv[1][0] == '1';
  const auto plan = legend_b200::plan_iteration_order(6);
  if (plan.state_offsets.size() != 9) return 2;  // n = 6 has 8 buffer states
  {  // host-only graph I/O: ingest a TSV, write and read back the reference's graph files
    const char* tsv = "binding_smoke_edges.tsv";
    if (FILE* f = std::fopen(tsv, "w")) {
      std::fputs("# src rel dst\n3 1 4\n1 0 5\n9 2 6\n", f);
      std::fclose(f);
    }
    const auto g = legend_b200::ingest_tsv(tsv, true);
    std::remove(tsv);
    if (g.edges.size() != 9 || g.num_nodes != 10 || g.num_relations != 3) return 6;
    legend_b200::write_graph("binding_smoke_graph", g.edges, g.num_nodes, g.num_relations);
    const auto back = legend_b200::read_graph("binding_smoke_graph");
    std::remove("binding_smoke_graph/edges.bin");
    std::remove("binding_smoke_graph/graph_meta.json");
    std::remove("binding_smoke_graph");
    if (back.edges != g.edges || back.num_nodes != 10) return 7;
    std::printf("graph io ok\n");
  }
  try {
    legend_b200::Trainer t({legend_b200::ScoreKind::kDistMult, 8}, {0.1, 1e-10, 64, 3, true, 7});
    std::vector<std::uint32_t> edges;
    for (std::uint32_t e = 0; e < 500; ++e) edges.insert(edges.end(), {e % 50, e % 3, (e * 7) % 50});
    t.set_graph(edges, 50, 3);
    t.make_partition_plan(4);
    t.init_store(42);
    const auto r = t.run_epoch(0);
    std::printf("epoch ok: %llu edges, loss %.6f\n", (unsigned long long)r.edges_trained, r.loss_sum);
    try {
      t.train_batch({0, 0, 99}, {1, 2, 3});
      return 3;
    } catch (const std::out_of_range&) {
    }
    return expect_gpu ? 0 : 4;
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error: %s\n", e.what());
    return expect_gpu ? 5 : 0;
  }
}
