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

// Multi-GPU partition-round schedule: rounds of disjoint
// partition pairs (circle method; odd n gets a bye per round).  Every bucket
// appears exactly once: (a,b) and (b,a) in the round pairing a and b, the
// diagonal (a,a) in the first round that holds a.  Buckets are numbered in
// one global order (round, pair, [diagonals], (a,b), (b,a)); that position
// keys the bucket's RNG stream, and the pair {a,b} is its negative pool, so
// the epoch is the same for any number of GPUs.  Pair j of a round runs on
// rank j % num_ranks.
struct RoundBucket {
  uint32_t src, dst;     // bucket (i, j)
  uint64_t g;            // global position (RNG stream index)
  uint32_t pool[2];      // the pair {a, b}, ascending (pool[1] = none for n = 1)
  uint32_t round, pair;
};
struct RoundSchedule {
  uint32_t n = 0;
  uint32_t num_rounds = 0;
  uint32_t pairs_per_round = 0;
  std::vector<RoundBucket> buckets;  // global order
};
RoundSchedule make_round_schedule(uint32_t n);

LoadingOrder make_loading_order(uint32_t n);
IterationPlan make_iteration_plan(const LoadingOrder& seq, uint32_t n);
IterationPlan single_state_plan(uint32_t n);

}  // namespace lgd
