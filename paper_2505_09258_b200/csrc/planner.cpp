// planner.cpp -- host side of the scheduler: the 3-slot buffer loading order
// and the bucket iteration order with prefetch points (ordering.hpp:49-54;
// PAPER.md Algorithms 1-2).  The epoch's RNG stream of bucket g is keyed by
// its position g in bucket_order (pipeline.cpp:296), so the plan must match
// the reference's exactly; tests/test_planner.py checks every n in 4..40
// against the reference library and the byte-stable fig6 fixture.
//
// make_loading_order / make_iteration_order are therefore a RESTATEMENT of
// the reference's plan_loading_order / plan_iteration_order
// (ordering.cpp:59-346), step for step (the column-owner sweep, the greedy
// swap choice, the seed prefix, the Kuhn matching for empty windows, and the
// same error texts): the bucket order is a bit-exact contract, not a design
// choice.  The multi-GPU round schedule (make_round_schedule) and the n <= 3
// single-state plan are new.
#include "planner.hpp"

#include <algorithm>
#include <stdexcept>

namespace lgd {

namespace {

struct Buffer {
  std::array<uint32_t, 3> slot;
  bool holds(uint32_t p) const { return slot[0] == p || slot[1] == p || slot[2] == p; }
};

// Pair coverage of the n x n bucket grid by the states seen so far.
class Coverage {
 public:
  explicit Coverage(uint32_t n) : n_(n), cell_(size_t(n) * n, 0), col_(n, 0) {}
  void add_state(const Buffer& b) {
    for (uint32_t x : b.slot)
      for (uint32_t y : b.slot) touch(x, y);
  }
  bool has(uint32_t x, uint32_t y) const { return cell_[size_t(x) * n_ + y] != 0; }
  bool column_full(uint32_t c) const { return col_[c] == n_; }
  bool complete() const { return filled_ == uint64_t(n_) * n_; }

 private:
  void touch(uint32_t x, uint32_t y) {
    uint8_t& c = cell_[size_t(x) * n_ + y];
    if (c) return;
    c = 1;
    ++col_[y];
    ++filled_;
  }
  uint32_t n_;
  std::vector<uint8_t> cell_;
  std::vector<uint32_t> col_;
  uint64_t filled_ = 0;
};

}  // namespace

// Column-separation order: after a rotation that sweeps every partition
// past partition 0, each "owner" column is completed in turn; the owner stays
// resident while the other two slots cycle through greedy loads.
LoadingOrder make_loading_order(uint32_t n) {
  if (n < 4) throw std::invalid_argument("loading order requires n >= 4");
  LoadingOrder seq;
  seq.n = n;
  Coverage cov(n);
  Buffer buf{{0, 1, 2}};
  seq.states.push_back(buf.slot);
  cov.add_state(buf);

  auto apply = [&](uint32_t out, uint32_t in) {
    for (auto& s : buf.slot) {
      if (s == out) {
        s = in;
        break;
      }
    }
    std::sort(buf.slot.begin(), buf.slot.end());
    seq.states.push_back(buf.slot);
    seq.swaps.push_back({out, in});
    cov.add_state(buf);
  };
  auto smallest_except = [&](uint32_t skip) {
    uint32_t best = kNoPartition;
    for (uint32_t s : buf.slot)
      if (s != skip && (best == kNoPartition || s < best)) best = s;
    return best;
  };

  for (uint32_t p = 3; p < n; ++p) apply(p - 2, p);  // sweep past partition 0

  uint32_t owner = 0;
  uint32_t cursor = n - 1;  // greedy scan starts after the last greedy load
  while (!cov.complete()) {
    uint32_t out = kNoPartition;
    if (cov.column_full(owner)) {
      const uint32_t next = owner + 1;
      if (buf.holds(next)) {
        owner = next;
        continue;
      }
      // keep loaded(k) != evicted(k+1): never evict what was just loaded
      const uint32_t leaving =
          (!seq.swaps.empty() && seq.swaps.back().loaded == owner) ? smallest_except(owner) : owner;
      apply(leaving, next);
      if (cov.complete()) break;
      out = smallest_except(next);
      owner = next;
    } else {
      const auto& before = seq.states[seq.states.size() - 2];
      const Buffer prev{before};
      for (uint32_t s : buf.slot) {
        if (s != owner && prev.holds(s)) {
          out = s;
          break;
        }
      }
      if (out == kNoPartition) throw std::logic_error("no eviction candidate");
    }
    uint32_t partner = kNoPartition;  // the resident that stays beside the owner
    for (uint32_t s : buf.slot)
      if (s != out && s != owner) partner = s;
    uint32_t pick = kNoPartition, pick_score = 0;
    for (uint32_t step = 1; step <= n; ++step) {
      const uint32_t cand = (cursor + step) % n;
      if (buf.holds(cand)) continue;
      const uint32_t score = (cov.has(cand, owner) ? 0u : 4u) +
                             (partner != kNoPartition && !cov.has(cand, partner) ? 1u : 0u);
      if (pick == kNoPartition || score > pick_score) {
        pick = cand;
        pick_score = score;
      }
    }
    if (pick == kNoPartition) throw std::logic_error("no load candidate");
    apply(out, pick);
    cursor = pick;
  }
  return seq;
}

namespace {

void check_sequence(const LoadingOrder& seq, uint32_t n) {
  if (seq.n != n) throw std::invalid_argument("sequence n mismatch");
  if (n < 4) throw std::invalid_argument("sequence requires n >= 4");
  if (seq.states.size() < 2) throw std::invalid_argument("sequence needs at least two states");
  if (seq.swaps.size() + 1 != seq.states.size())
    throw std::invalid_argument("swap list inconsistent with state list");
  for (const auto& s : seq.states)
    if (!(s[0] < s[1] && s[1] < s[2]) || s[2] >= n)
      throw std::invalid_argument("buffer state must hold 3 distinct sorted partition ids");
  for (size_t i = 0; i + 1 < seq.states.size(); ++i) {
    const Buffer cur{seq.states[i]};
    const auto& sw = seq.swaps[i];
    if (!cur.holds(sw.evicted) || cur.holds(sw.loaded))
      throw std::invalid_argument("swap does not apply to its state");
    auto next = seq.states[i];
    for (auto& s : next)
      if (s == sw.evicted) s = sw.loaded;
    std::sort(next.begin(), next.end());
    if (next != seq.states[i + 1])
      throw std::invalid_argument("consecutive states must differ by exactly the recorded swap");
  }
}

// Bipartite matching of non-final states to buckets they can compute while
// their swap is in flight (the 4 buckets not touching the evictee), so that
// every overlap window is non-empty.  Augmenting paths, candidates in
// ascending bucket-id order.
class WindowMatcher {
 public:
  WindowMatcher(const LoadingOrder& seq, uint32_t n)
      : seq_(seq), n_(n), owner_(size_t(n) * n, kUnset), seen_(size_t(n) * n, 0) {}
  void fix(uint32_t bucket, size_t state) { owner_[bucket] = state; }
  bool place(size_t state) {
    std::fill(seen_.begin(), seen_.end(), 0);
    return augment(state);
  }
  size_t owner(uint32_t bucket) const { return owner_[bucket]; }
  static constexpr size_t kUnset = ~size_t(0);

 private:
  std::vector<uint32_t> options(size_t state) const {
    const uint32_t ev = seq_.swaps[state].evicted;
    std::vector<uint32_t> out;
    for (uint32_t a : seq_.states[state])
      for (uint32_t b : seq_.states[state])
        if (a != ev && b != ev) out.push_back(a * n_ + b);
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    return out;
  }
  bool augment(size_t state) {
    for (uint32_t b : options(state)) {
      if (seen_[b]) continue;
      seen_[b] = 1;
      if (owner_[b] == kUnset || augment(owner_[b])) {
        owner_[b] = state;
        return true;
      }
    }
    return false;
  }
  const LoadingOrder& seq_;
  uint32_t n_;
  std::vector<size_t> owner_;
  std::vector<uint8_t> seen_;
};

}  // namespace

IterationPlan make_iteration_plan(const LoadingOrder& seq, uint32_t n) {
  check_sequence(seq, n);
  if (seq.states[0] != std::array<uint32_t, 3>{0, 1, 2} || seq.swaps[0].evicted != 1)
    throw std::invalid_argument("iteration order expects initial state {0,1,2} evicting 1");
  const size_t S = seq.states.size();
  constexpr size_t kUnplaced = ~size_t(0);

  // Eager placement: each bucket goes to the first state holding both
  // endpoints -- evictee-related buckets first, then the overlap window.
  std::vector<std::vector<uint32_t>> early(S), window(S);
  std::vector<size_t> home(size_t(n) * n, kUnplaced);
  auto place = [&](size_t st, uint32_t a, uint32_t b, bool in_window) {
    const uint32_t id = a * n + b;
    if (home[id] != kUnplaced) return;
    home[id] = st;
    (in_window ? window : early)[st].push_back(id);
  };
  for (size_t i = 0; i < S; ++i) {
    const auto& st = seq.states[i];
    if (i + 1 == S) {
      for (uint32_t a : st)
        for (uint32_t b : st) place(i, a, b, true);
      continue;
    }
    const uint32_t ev = seq.swaps[i].evicted;
    if (i == 0) {
      const uint32_t seed_prefix[5][2] = {{0, 1}, {1, 1}, {1, 0}, {1, 2}, {2, 1}};
      for (const auto& pr : seed_prefix) place(0, pr[0], pr[1], false);
    } else {
      const uint32_t fresh = seq.swaps[i - 1].loaded;
      for (uint32_t x : st) {
        if (x == fresh) continue;
        place(i, ev, x, false);
        if (x != ev) place(i, x, ev, false);
      }
      if (Buffer{st}.holds(fresh)) {
        place(i, ev, fresh, false);
        if (fresh != ev) place(i, fresh, ev, false);
      }
    }
    for (uint32_t a : st)
      for (uint32_t b : st)
        if (a != ev && b != ev) place(i, a, b, true);
  }
  for (size_t h : home)
    if (h == kUnplaced) throw std::invalid_argument("sequence does not cover all partition pairs");

  WindowMatcher match(seq, n);
  for (size_t i = 0; i + 1 < S; ++i)
    if (!window[i].empty()) match.fix(window[i][0], i);
  for (size_t i = 0; i + 1 < S; ++i)
    if (window[i].empty() && !match.place(i))
      throw std::logic_error("no bucket available to keep the overlap window non-empty");
  // Move matched buckets into their state's window.  Every state receives at
  // most one bucket, so the visiting order does not change the result.
  for (uint32_t id = 0; id < n * n; ++id) {
    const size_t to = match.owner(id);
    if (to == WindowMatcher::kUnset || to == home[id]) continue;
    auto erase = [&](std::vector<uint32_t>& v) { v.erase(std::remove(v.begin(), v.end(), id), v.end()); };
    erase(early[home[id]]);
    erase(window[home[id]]);
    window[to].push_back(id);
    home[id] = to;
  }

  IterationPlan plan;
  plan.seq = seq;
  for (size_t i = 0; i < S; ++i) {
    plan.state_offsets.push_back(plan.bucket_order.size());
    for (uint32_t id : early[i]) plan.bucket_order.push_back({id / n, id % n});
    if (i + 1 < S) plan.prefetch_points.push_back(plan.bucket_order.size());
    for (uint32_t id : window[i]) plan.bucket_order.push_back({id / n, id % n});
  }
  plan.state_offsets.push_back(plan.bucket_order.size());
  return plan;
}

RoundSchedule make_round_schedule(uint32_t n) {
  if (n < 1) throw std::invalid_argument("partition count must be >= 1");
  RoundSchedule rs;
  rs.n = n;
  if (n == 1) {
    rs.num_rounds = 1;
    rs.pairs_per_round = 1;
    rs.buckets.push_back({0, 0, 0, {0, kNoPartition}, 0, 0});
    return rs;
  }
  const uint32_t m = n + (n & 1);  // even player count; player n (odd n) is the bye
  rs.num_rounds = m - 1;
  rs.pairs_per_round = m / 2;
  std::vector<uint8_t> diag_done(n, 0);
  uint64_t g = 0;
  for (uint32_t r = 0; r < m - 1; ++r) {
    // circle method: player m-1 fixed, the others rotate
    std::vector<std::pair<uint32_t, uint32_t>> pairs;
    pairs.push_back({r, m - 1});
    for (uint32_t i = 1; i < m / 2; ++i)
      pairs.push_back({(r + i) % (m - 1), (r + m - 1 - i) % (m - 1)});
    uint32_t j = 0;
    for (auto [x, y] : pairs) {
      const uint32_t a = std::min(x, y), b = std::max(x, y);
      if (b >= n) {  // bye: a still gets its diagonal when first seen
        if (!diag_done[a]) {
          diag_done[a] = 1;
          rs.buckets.push_back({a, a, g++, {a, kNoPartition}, r, j});
        }
        ++j;
        continue;
      }
      const uint32_t pool[2] = {a, b};
      for (uint32_t q : {a, b}) {
        if (!diag_done[q]) {
          diag_done[q] = 1;
          rs.buckets.push_back({q, q, g++, {pool[0], pool[1]}, r, j});
        }
      }
      rs.buckets.push_back({a, b, g++, {pool[0], pool[1]}, r, j});
      rs.buckets.push_back({b, a, g++, {pool[0], pool[1]}, r, j});
      ++j;
    }
  }
  return rs;
}

IterationPlan single_state_plan(uint32_t n) {
  if (n < 1 || n > 3) throw std::invalid_argument("single-state plan is for n <= 3");
  IterationPlan plan;
  plan.seq.n = n;
  std::array<uint32_t, 3> st{kNoPartition, kNoPartition, kNoPartition};
  for (uint32_t p = 0; p < n; ++p) st[p] = p;
  plan.seq.states.push_back(st);
  for (uint32_t a = 0; a < n; ++a)
    for (uint32_t b = 0; b < n; ++b) plan.bucket_order.push_back({a, b});
  plan.state_offsets = {0, uint64_t(n) * n};
  return plan;
}

}  // namespace lgd
