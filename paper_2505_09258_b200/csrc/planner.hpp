// planner.hpp -- host scheduler types (BufferStateSequence / IterationPlan,
// ordering.hpp:15-47).
#pragma once

#include <array>
#include <cstdint>
#include <utility>
#include <vector>

namespace lgd {

constexpr uint32_t kNoPartition = 0xffffffffu;

struct Swap {
  uint32_t evicted;
  uint32_t loaded;
};

struct LoadingOrder {
  uint32_t n = 0;
  std::vector<std::array<uint32_t, 3>> states;  // sorted ascending
  std::vector<Swap> swaps;                      // states.size() - 1
};

struct IterationPlan {
  LoadingOrder seq;
  std::vector<std::pair<uint32_t, uint32_t>> bucket_order;  // n*n buckets
  std::vector<uint64_t> state_offsets;                      // states + 1
  std::vector<uint64_t> prefetch_points;                    // states - 1
};

LoadingOrder make_loading_order(uint32_t n);
IterationPlan make_iteration_plan(const LoadingOrder& seq, uint32_t n);
IterationPlan single_state_plan(uint32_t n);

}  // namespace lgd
