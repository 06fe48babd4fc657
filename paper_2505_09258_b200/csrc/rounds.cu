// rounds.cu -- the multi-GPU partition-round runner (SURVEY.md
// 8(e)): one process per GPU, host C++ behind the C ABI.
//
// Schedule (planner.cpp make_round_schedule): rounds of disjoint partition
// pairs, every bucket once, its global position g keying its RNG stream
// (pipeline.cpp:296) and its pair {a, b} the negative pool; pair j of a round
// runs on rank j % world.  Ranks own disjoint partitions within a round, so
// node updates never conflict.  Every rank allocates the full tables (all
// configured graphs fit one B200); a partition's rows are current only on
// the rank that last trained it, and move to the next user between rounds.
//
// Hand-offs ride NVLink as pulls on a side stream, overlapped with compute
// (Legend's prefetch, moved onto peer copies):
//   * after its last bucket touching partition p in round r, the holder
//     records an inter-process event ready[p] on its training stream;
//   * once every rank has QUEUED round r (a host barrier on a control NCCL
//     communicator -- no device work waits for it), the next holder's copy
//     stream waits on the peer's ready[p] and copies p's theta / state rows
//     from the peer's table (CUDA IPC mapping, cudaMemcpyPeerAsync) into its
//     own, then records arrived[p];
//   * the next holder's training stream waits on arrived[p] only before its
//     first bucket touching p.
// So a partition moves while both ranks still train their other buckets:
// whenever a rank holds several pairs in a round (world < n / 2), the first
// pair's partitions stream out during the second pair's buckets.  With one
// pair per rank every bucket touches both partitions and the copy is exposed
// (~3 ms for a 2.1 GB TW partition at NVLink rates vs ~135 ms of compute).
//
// Typed models share the relation table: ranks run their batches in lock step
// and sum the dense relation gradients [R x (d+1)] with ncclAllReduce on the
// training stream (stream-ordered: no host round trip per batch); every rank
// applies the identical Adagrad step.  Batch counts of every rank are known
// from the partition plan, so the lock-step length needs no collective.
//
// NCCL is loaded at run time (dlopen libnccl.so.2; torch's copy when torch
// already loaded it), so single-GPU use never needs it.  Virtual ranks (one
// context per rank in one process, lgd_comm_init_local) share events and
// table pointers directly; their caller runs every rank's enqueue before any
// hand-off (the 1-GPU test harness).
#include <dlfcn.h>
#include <nccl.h>

#include <memory>

#include "context.hpp"

namespace lgd {

namespace {

// ------------------------------------------------------------------ NCCL
struct Nccl {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static Nccl& get() {
    static Nccl n;
    if (!n.lib) {
      n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!n.lib) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
      auto sym = [&](const char* name) {
        void* f = dlsym(n.lib, name);
        if (!f) throw std::runtime_error(std::string("libnccl.so.2 lacks ") + name);
        return f;
      };
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
      n.CommSplit = reinterpret_cast<decltype(n.CommSplit)>(sym("ncclCommSplit"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
      n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
      n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    }
    return n;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw std::runtime_error(std::string(what) + ": " + (GetErrorString ? GetErrorString(r) : "NCCL error"));
  }
};

}  // namespace

// ------------------------------------------------------- host round plan
// The per-rank view of the schedule: which buckets, in which order, which
// partitions arrive before the round (from which rank) and which leave after
// it.  Pure host logic (lgd_round_actions exports it for the CPU tests).
struct RankRound {
  std::vector<size_t> items;                      // indices into sched.buckets, global order
  std::vector<std::pair<uint32_t, int>> arrive;   // (partition, from rank) before the round
  std::vector<uint32_t> depart;                   // partitions another rank uses next
};

static int pair_rank(uint32_t pair, uint32_t world) { return (int)(pair % world); }

// users[r][p] = rank that trains on partition p in round r (-1: none)
static std::vector<std::vector<int>> round_users(const RoundSchedule& rs, uint32_t world) {
  std::vector<std::vector<int>> u(rs.num_rounds, std::vector<int>(rs.n, -1));
  for (const auto& b : rs.buckets)
    for (uint32_t p : b.pool)
      if (p != kNoPartition) u[b.round][p] = pair_rank(b.pair, world);
  return u;
}

// `owner`: partition -> rank holding its current rows (-1: identical on all
// ranks, the state after lgd_init_store / lgd_load_partition on every rank)
static RankRound rank_round(const RoundSchedule& rs, const std::vector<std::vector<int>>& users,
                            uint32_t world, uint32_t rank, uint32_t r,
                            const std::vector<int>& owner) {
  RankRound rr;
  for (size_t i = 0; i < rs.buckets.size(); ++i)
    if (rs.buckets[i].round == r && pair_rank(rs.buckets[i].pair, world) == (int)rank)
      rr.items.push_back(i);
  for (uint32_t p = 0; p < rs.n; ++p) {
    if (users[r][p] == (int)rank && owner[p] >= 0 && owner[p] != (int)rank)
      rr.arrive.push_back({p, owner[p]});
    const uint32_t nr = (r + 1) % rs.num_rounds;  // the next round (next epoch after the last)
    if (users[r][p] == (int)rank && users[nr][p] >= 0 && users[nr][p] != (int)rank)
      rr.depart.push_back(p);
  }
  return rr;
}

// ------------------------------------------------------------ the runner
struct RoundRunner {
  lgd_context* ctx = nullptr;
  uint32_t world = 1, rank = 0;
  RoundSchedule sched;
  std::vector<std::vector<int>> users;
  std::vector<int> owner;  // partition -> rank with its current rows (-1: all)
  bool local = false;      // virtual ranks in one process
  bool use_nccl = false;   // NCCL communicators (every multi-process run; optional at world 1)
  // NCCL (multi-process)
  ncclComm_t data = nullptr, ctrl = nullptr;
  cudaStream_t ctrl_stream = nullptr;
  DevBuf<int> barrier_buf;
  // hand-offs
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> ready;    // own, per partition (inter-process)
  std::vector<cudaEvent_t> arrived;  // own, per partition
  std::vector<char> arrival_pending;
  std::vector<std::vector<cudaEvent_t>> peer_ready;  // [rank][p]
  std::vector<float*> peer_theta, peer_state;        // [rank]
  std::vector<bool> peer_mapped;
  cudaEvent_t h0 = nullptr, h1 = nullptr;
  bool handoff_timed = false;
  uint64_t handoff_bytes = 0;
  // the queued round
  bool queued = false;
  uint32_t q_epoch = 0, q_round = 0;
  RankRound q;
  bool lock_step = false;
  DevBuf<double> rel_buf;
  float* theta_at_init = nullptr;

  ~RoundRunner() {
    cudaSetDevice(ctx->device);
    if (copy) cudaStreamSynchronize(copy);
    for (size_t q2 = 0; q2 < peer_theta.size(); ++q2) {
      if (!local && peer_mapped[q2]) {
        cudaIpcCloseMemHandle(peer_theta[q2]);
        cudaIpcCloseMemHandle(peer_state[q2]);
      }
      if (!local && q2 != rank)
        for (auto e : peer_ready[q2]) cudaEventDestroy(e);
    }
    for (auto e : ready) cudaEventDestroy(e);
    for (auto e : arrived) cudaEventDestroy(e);
    if (h0) cudaEventDestroy(h0);
    if (h1) cudaEventDestroy(h1);
    if (copy) cudaStreamDestroy(copy);
    if (ctrl_stream) cudaStreamDestroy(ctrl_stream);
    if (data || ctrl) {
      Nccl& n = Nccl::get();
      if (ctrl) n.CommDestroy(ctrl);
      if (data) n.CommDestroy(data);
    }
  }

  void setup_common(lgd_context* c, uint32_t r, uint32_t w) {
    ctx = c;
    rank = r;
    world = w;
    if (!c->partitioned) throw std::invalid_argument("no partition plan");
    if (!c->tables_ready) throw std::invalid_argument("embedding store not initialised");
    sched = make_round_schedule(c->n);
    users = round_users(sched, world);
    owner.assign(c->n, -1);
    theta_at_init = c->theta.get();
    LGD_CUDA(cudaStreamCreateWithPriority(&copy, cudaStreamNonBlocking, 0));
    ready.resize(c->n);
    arrived.resize(c->n);
    arrival_pending.assign(c->n, 0);
    for (uint32_t p = 0; p < c->n; ++p) {
      LGD_CUDA(cudaEventCreateWithFlags(&ready[p], cudaEventDisableTiming |
                                                       (use_nccl && !local ? cudaEventInterprocess : 0)));
      LGD_CUDA(cudaEventCreateWithFlags(&arrived[p], cudaEventDisableTiming));
    }
    LGD_CUDA(cudaEventCreate(&h0));
    LGD_CUDA(cudaEventCreate(&h1));
    peer_theta.assign(w, nullptr);
    peer_state.assign(w, nullptr);
    peer_mapped.assign(w, false);
    peer_ready.assign(w, {});
    // typed models sum relation gradients per lock-step batch over NCCL (also
    // at world 1 when the communicators exist: a one-rank all-reduce)
    lock_step = c->typed() && c->R && (w > 1 || (use_nccl && !local));
    if (lock_step && local) throw std::invalid_argument("virtual ranks: typed models need the lock-step primitives (lgd_round_step)");
    if (lock_step) rel_buf.reserve(c->R * (c->dim + 1));
  }

  // multi-process: NCCL data + control communicators, IPC table / event maps
  void setup_nccl(const void* id) {
    Nccl& n = Nccl::get();
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    n.check(n.CommInitRank(&data, (int)world, uid, (int)rank), "ncclCommInitRank");
    n.check(n.CommSplit(data, 0, (int)rank, &ctrl, nullptr), "ncclCommSplit");
    LGD_CUDA(cudaStreamCreateWithFlags(&ctrl_stream, cudaStreamNonBlocking));
    barrier_buf.reserve(1);
    // every rank's table handles and ready events, gathered over the control comm
    const uint32_t np = ctx->n;
    const size_t blob = 2 * sizeof(cudaIpcMemHandle_t) + np * sizeof(cudaIpcEventHandle_t);
    std::vector<char> mine(blob), all(blob * world);
    cudaIpcMemHandle_t mh;
    LGD_CUDA(cudaIpcGetMemHandle(&mh, ctx->theta.get()));
    std::memcpy(mine.data(), &mh, sizeof mh);
    LGD_CUDA(cudaIpcGetMemHandle(&mh, ctx->state.get()));
    std::memcpy(mine.data() + sizeof mh, &mh, sizeof mh);
    for (uint32_t p = 0; p < np; ++p) {
      cudaIpcEventHandle_t eh;
      LGD_CUDA(cudaIpcGetEventHandle(&eh, ready[p]));
      std::memcpy(mine.data() + 2 * sizeof mh + p * sizeof eh, &eh, sizeof eh);
    }
    DevBuf<char> dmine, dall;
    dmine.reserve(blob);
    dall.reserve(blob * world);
    LGD_CUDA(cudaMemcpy(dmine.get(), mine.data(), blob, cudaMemcpyHostToDevice));
    n.check(n.AllGather(dmine.get(), dall.get(), blob, ncclChar, ctrl, ctrl_stream), "ncclAllGather");
    LGD_CUDA(cudaStreamSynchronize(ctrl_stream));
    LGD_CUDA(cudaMemcpy(all.data(), dall.get(), blob * world, cudaMemcpyDeviceToHost));
    for (uint32_t q2 = 0; q2 < world; ++q2) {
      if (q2 == rank) {
        peer_theta[q2] = ctx->theta.get();
        peer_state[q2] = ctx->state.get();
        peer_ready[q2] = ready;
        continue;
      }
      const char* b = all.data() + q2 * blob;
      void* pt = nullptr;
      void* ps = nullptr;
      std::memcpy(&mh, b, sizeof mh);
      LGD_CUDA(cudaIpcOpenMemHandle(&pt, mh, cudaIpcMemLazyEnablePeerAccess));
      std::memcpy(&mh, b + sizeof mh, sizeof mh);
      LGD_CUDA(cudaIpcOpenMemHandle(&ps, mh, cudaIpcMemLazyEnablePeerAccess));
      peer_theta[q2] = static_cast<float*>(pt);
      peer_state[q2] = static_cast<float*>(ps);
      peer_mapped[q2] = true;
      peer_ready[q2].resize(np);
      for (uint32_t p = 0; p < np; ++p) {
        cudaIpcEventHandle_t eh;
        std::memcpy(&eh, b + 2 * sizeof mh + p * sizeof eh, sizeof eh);
        LGD_CUDA(cudaIpcOpenEventHandle(&peer_ready[q2][p], eh));
      }
    }
    barrier();
  }

  // host barrier: returns once every rank got here (control comm, its own
  // stream -- no training work is waited for)
  void barrier() {
    if (world == 1 || local) return;
    Nccl& n = Nccl::get();
    n.check(n.AllReduce(barrier_buf.get(), barrier_buf.get(), 1, ncclInt32, ncclSum, ctrl,
                        ctrl_stream),
            "ncclAllReduce (barrier)");
    LGD_CUDA(cudaStreamSynchronize(ctrl_stream));
  }

  void check_tables() const {
    if (ctx->theta.get() != theta_at_init)
      throw std::logic_error("tables were reallocated after lgd_comm_init");
  }

  bool touches(size_t item, uint32_t p) const {
    const auto& b = sched.buckets[item];
    return b.src == p || b.dst == p;
  }

  // queue this rank's round r: arrivals waited on before the first bucket
  // touching them, ready[p] recorded after the last bucket touching a
  // departing partition
  void enqueue(uint32_t epoch, uint32_t r) {
    if (queued) throw std::logic_error("previous round not collected");
    if (r >= sched.num_rounds) throw std::invalid_argument("round out of range");
    check_tables();
    q = rank_round(sched, users, world, rank, r, owner);
    std::vector<lgd_context::WorkItem> items;
    for (size_t i : q.items) {
      const auto& b = sched.buckets[i];
      const uint32_t pool[3] = {b.pool[0], b.pool[1], kNoPartition};
      items.push_back({b.src, b.dst, b.g, ctx->pool_of_parts(pool, 3)});
    }
    // first / last local item touching each partition
    const uint32_t np = ctx->n;
    std::vector<long> first(np, -1), last(np, -1);
    for (size_t j = 0; j < q.items.size(); ++j)
      for (uint32_t p : {sched.buckets[q.items[j]].src, sched.buckets[q.items[j]].dst}) {
        if (first[p] < 0) first[p] = (long)j;
        last[p] = (long)j;
      }
    std::vector<char> departs(np, 0);
    for (uint32_t p : q.depart) departs[p] = 1;
    auto hook = [&](size_t j, bool before) {
      for (uint32_t p : {sched.buckets[q.items[j]].src, sched.buckets[q.items[j]].dst}) {
        if (before && first[p] == (long)j && arrival_pending[p]) {
          LGD_CUDA(cudaStreamWaitEvent(ctx->stream, arrived[p], 0));
          arrival_pending[p] = 0;
        }
        if (!before && last[p] == (long)j && departs[p]) {
          LGD_CUDA(cudaEventRecord(ready[p], ctx->stream));
          departs[p] = 0;
        }
      }
    };
    // arrivals no bucket of ours touches (cannot happen in the pair schedule)
    for (auto [p, from] : q.arrive)
      if (first[p] < 0 && arrival_pending[p]) {
        LGD_CUDA(cudaStreamWaitEvent(ctx->stream, arrived[p], 0));
        arrival_pending[p] = 0;
      }
    const std::function<void(size_t, bool)> fn = hook;
    if (!lock_step) {
      ctx->train_items(epoch, items, nullptr, ctx->host_edges, ~uint64_t(0), nullptr, &fn, false);
    } else {
      // lock step: every rank's batch count follows from the partition plan
      uint64_t steps = 0;
      for (uint32_t q2 = 0; q2 < world; ++q2) {
        uint64_t nb = 0;
        for (size_t i = 0; i < sched.buckets.size(); ++i) {
          const auto& b = sched.buckets[i];
          if (b.round != r || pair_rank(b.pair, world) != (int)q2) continue;
          const uint64_t bi = uint64_t(b.src) * ctx->n + b.dst;
          nb += (ctx->offsets[bi + 1] - ctx->offsets[bi] + ctx->opt.batch_size - 1) / ctx->opt.batch_size;
        }
        steps = std::max(steps, nb);
      }
      const uint64_t mine = ctx->round_begin(epoch, items);
      const auto& fb = ctx->round_first_batch;  // per item, prefix of batch counts
      const bool was_ordered = ctx->stream_ordered;
      ctx->stream_ordered = true;
      Nccl& n = Nccl::get();
      size_t next_before = 0, next_after = 0;
      for (uint64_t s = 0; s < steps; ++s) {
        while (next_before < items.size() && fb[next_before] <= s) fn(next_before++, true);
        ctx->round_step(s, rel_buf.get());
        n.check(n.AllReduce(rel_buf.get(), rel_buf.get(), ctx->R * (ctx->dim + 1), ncclFloat64,
                            ncclSum, data, ctx->stream),
                "ncclAllReduce (relations)");
        ctx->round_apply_relations(rel_buf.get());
        while (next_after < next_before && fb[next_after + 1] <= s + 1) fn(next_after++, false);
      }
      (void)mine;
      while (next_before < items.size()) fn(next_before++, true);
      while (next_after < items.size()) fn(next_after++, false);
      ctx->stream_ordered = was_ordered;
    }
    q_epoch = epoch;
    q_round = r;
    queued = true;
  }

  // once every rank queued its round: pull the next round's arrivals
  void handoff() {
    if (!queued) throw std::logic_error("no queued round");
    barrier();
    const uint32_t nr = (q_round + 1) % sched.num_rounds;
    // the next round's holders; ownership after this round
    std::vector<int> after = owner;
    for (uint32_t p = 0; p < ctx->n; ++p)
      if (users[q_round][p] >= 0) after[p] = users[q_round][p];
    handoff_bytes = 0;
    handoff_timed = false;
    for (uint32_t p = 0; p < ctx->n; ++p) {
      const int from = after[p];
      if (users[nr][p] != (int)rank || from < 0 || from == (int)rank) continue;
      const uint64_t off = ctx->part_begin(p) * ctx->dim, cnt = ctx->part_rows(p) * ctx->dim;
      if (!handoff_timed) LGD_CUDA(cudaEventRecord(h0, copy));
      handoff_timed = true;
      LGD_CUDA(cudaStreamWaitEvent(copy, peer_ready[from][p], 0));
      LGD_CUDA(cudaMemcpyAsync(ctx->theta.get() + off, peer_theta[from] + off, cnt * 4,
                               cudaMemcpyDefault, copy));
      LGD_CUDA(cudaMemcpyAsync(ctx->state.get() + off, peer_state[from] + off, cnt * 4,
                               cudaMemcpyDefault, copy));
      LGD_CUDA(cudaEventRecord(arrived[p], copy));
      arrival_pending[p] = 1;
      handoff_bytes += 8 * cnt;
    }
    if (handoff_timed) LGD_CUDA(cudaEventRecord(h1, copy));
    owner = after;
  }

  void collect(lgd_epoch_result* out, double* handoff_ms, uint64_t* bytes) {
    if (!queued) throw std::logic_error("no queued round");
    if (!lock_step)
      ctx->finish_items(out);
    else
      ctx->round_end(out);
    float ms = 0;
    if (handoff_timed) {
      LGD_CUDA(cudaEventSynchronize(h1));
      LGD_CUDA(cudaEventElapsedTime(&ms, h0, h1));
    }
    if (handoff_ms) *handoff_ms = ms;
    if (bytes) *bytes = handoff_bytes;
    queued = false;
  }
};

void destroy_round_runner(RoundRunner* r) { delete r; }

}  // namespace lgd

// ============================================================== C ABI ====
extern "C" {

int lgd_comm_unique_id(void* id128) {
  return guarded([&] {
    if (!id128) throw std::invalid_argument("null argument");
    Nccl& n = Nccl::get();
    ncclUniqueId uid;
    n.check(n.GetUniqueId(&uid), "ncclGetUniqueId");
    std::memcpy(id128, &uid, sizeof uid);
  });
}

int lgd_comm_init(lgd_context* ctx, const void* id128, uint32_t rank, uint32_t world) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (world == 0 || rank >= world) throw std::invalid_argument("rank out of range");
    if (world > 1 && !id128) throw std::invalid_argument("null NCCL id");
    DeviceGuard g(ctx->device);
    ctx->wait_stores();
    ctx->runner.reset();
    auto r = std::make_unique<RoundRunner>();
    // an id means NCCL communicators, also at world 1 (a one-rank check of the
    // NCCL / IPC set-up); no id at world 1: a single process without NCCL
    r->use_nccl = id128 != nullptr;
    r->setup_common(ctx, rank, world);
    if (r->use_nccl) r->setup_nccl(id128);
    ctx->runner.reset(r.release());
  });
}

int lgd_comm_init_local(lgd_context** ctxs, uint32_t world) {
  return guarded([&] {
    if (!ctxs || world == 0) throw std::invalid_argument("null argument");
    for (uint32_t q = 0; q < world; ++q) {
      if (!ctxs[q]) throw std::invalid_argument("null context");
      if (ctxs[q]->n != ctxs[0]->n) throw std::invalid_argument("contexts differ in partitions");
    }
    for (uint32_t q = 0; q < world; ++q) {
      DeviceGuard g(ctxs[q]->device);
      ctxs[q]->wait_stores();
      ctxs[q]->runner.reset();
      auto r = std::make_unique<RoundRunner>();
      r->local = true;
      r->setup_common(ctxs[q], q, world);
      ctxs[q]->runner.reset(r.release());
    }
    for (uint32_t q = 0; q < world; ++q)
      for (uint32_t q2 = 0; q2 < world; ++q2) {
        RoundRunner* r = ctxs[q]->runner.get();
        r->peer_theta[q2] = ctxs[q2]->theta.get();
        r->peer_state[q2] = ctxs[q2]->state.get();
        r->peer_ready[q2] = ctxs[q2]->runner->ready;
      }
  });
}

int lgd_round_enqueue(lgd_context* ctx, uint32_t epoch, uint32_t round) {
  return guarded([&] {
    if (!ctx) throw std::invalid_argument("null context");
    if (!ctx->runner) throw std::logic_error("lgd_comm_init first");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->runner->enqueue(epoch, round);
  });
}

int lgd_round_handoff(lgd_context* ctx) {
  return guarded([&] {
    if (!ctx || !ctx->runner) throw std::logic_error("lgd_comm_init first");
    DeviceGuard g(ctx->device);
    ctx->runner->handoff();
  });
}

int lgd_round_collect(lgd_context* ctx, lgd_epoch_result* out, double* handoff_ms,
                      uint64_t* handoff_bytes) {
  return guarded([&] {
    if (!ctx || !ctx->runner) throw std::logic_error("lgd_comm_init first");
    DeviceGuard g(ctx->device);
    ctx->runner->collect(out, handoff_ms, handoff_bytes);
  });
}

int lgd_train_round(lgd_context* ctx, uint32_t epoch, uint32_t round, lgd_epoch_result* out,
                    double* handoff_ms, uint64_t* handoff_bytes) {
  return guarded([&] {
    if (!ctx || !ctx->runner) throw std::logic_error("lgd_comm_init first");
    if (ctx->runner->local && ctx->runner->world > 1)
      throw std::logic_error("virtual ranks: enqueue every rank before any hand-off");
    DeviceGuard g(ctx->device);
    ctx->fence_stores();
    ctx->runner->enqueue(epoch, round);
    ctx->runner->handoff();
    ctx->runner->collect(out, handoff_ms, handoff_bytes);
  });
}

int lgd_round_count(lgd_context* ctx, uint32_t* rounds) {
  return guarded([&] {
    if (!ctx || !ctx->runner || !rounds) throw std::logic_error("lgd_comm_init first");
    *rounds = ctx->runner->sched.num_rounds;
  });
}

int lgd_round_actions(uint32_t n, uint32_t world, uint32_t rank, uint32_t round,
                      const int32_t* owner_in, uint64_t capacity, uint64_t* count,
                      lgd_round_action* out, int32_t* owner_out) {
  return guarded([&] {
    if (!count) throw std::invalid_argument("null argument");
    if (world == 0 || rank >= world) throw std::invalid_argument("rank out of range");
    const RoundSchedule rs = make_round_schedule(n);
    if (round >= rs.num_rounds) throw std::invalid_argument("round out of range");
    const auto users = round_users(rs, world);
    std::vector<int> owner(n, -1);
    if (owner_in)
      for (uint32_t p = 0; p < n; ++p) owner[p] = owner_in[p];
    const RankRound rr = rank_round(rs, users, world, rank, round, owner);
    std::vector<lgd_round_action> acts;
    for (auto [p, from] : rr.arrive) acts.push_back({LGD_ACT_ARRIVE, p, from, 0});
    for (size_t i : rr.items) acts.push_back({LGD_ACT_TRAIN, kNoPartition, -1, (uint64_t)i});
    const uint32_t nr = (round + 1) % rs.num_rounds;
    for (uint32_t p : rr.depart) acts.push_back({LGD_ACT_DEPART, p, users[nr][p], 0});
    *count = acts.size();
    if (out)
      for (size_t i = 0; i < acts.size() && i < capacity; ++i) out[i] = acts[i];
    if (owner_out) {
      for (uint32_t p = 0; p < n; ++p)
        owner_out[p] = users[round][p] >= 0 ? users[round][p] : owner[p];
    }
  });
}

}  // extern "C"
