"""Multi-GPU partition-round scheduler.

Exact reference semantics do not shard: batches are sequentially dependent
and every batch samples negatives from all three resident partitions.  The
multi-GPU epoch is therefore a *schedule* with its own, stated semantics,
rebuilt from the reference primitives and checked against a serialised CPU
restatement (oracle ``run_rounds``):

* rounds of disjoint partition pairs (circle method), every bucket once, in
  one global order whose position keys the bucket's RNG stream
  (``derive_seed(seed, "bukt", epoch, g)``, pipeline.cpp:296);
* a bucket's negative pool is its pair {a, b};
* pair j of a round runs on rank ``j % world``; ranks own disjoint
  partitions within a round, so node updates never conflict;
* typed models share the relation table: ranks run their batches in lock
  step, the dense relation gradients [R x (d+1)] are summed across ranks
  (NCCL all-reduce) and every rank applies the same Adagrad step;
* between rounds each partition moves from its previous owner to its next
  one (NCCL send/recv over NVLink); tables are allocated on every rank so a
  hand-off is a plain row-range copy.

The driver below is communicator-agnostic: ``DistComm`` wraps
``torch.distributed`` (NCCL on GPUs, gloo in the CPU tests) and
``run_epoch_virtual`` steps several trainers in one process (the 1-GPU
parity test).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import legend as L

ITEM_DTYPE = np.dtype([("src", "<u4"), ("dst", "<u4"), ("g", "<u8"), ("pool", "<u4", (3,)),
                       ("round", "<u4"), ("pair", "<u4"), ("_pad", "<u4")])
assert ITEM_DTYPE.itemsize == 40


def round_schedule(n: int) -> np.ndarray:
    """The global bucket schedule (lgd_round_schedule) as a structured array."""
    lib = L.library()
    cnt = np.zeros(1, np.uint64)
    L._check(lib.lgd_round_schedule(n, 0, L._p(cnt), None, None, None))
    items = np.zeros(int(cnt[0]), ITEM_DTYPE)
    L._check(lib.lgd_round_schedule(n, len(items), L._p(cnt), items.ctypes.data_as(C.c_void_p),
                                    None, None))
    return items


ACTION_DTYPE = np.dtype([("kind", "<u4"), ("part", "<u4"), ("peer", "<i4"), ("_pad", "<u4"),
                         ("item", "<u8")])
assert ACTION_DTYPE.itemsize == 24
ARRIVE, TRAIN, DEPART = 0, 1, 2


def round_actions(n: int, world: int, rank: int, r: int, owner=None):
    """The C++ runner's plan for one rank and round (lgd_round_actions, host
    only): ARRIVE (partition, from peer) before the round, TRAIN buckets
    (index into round_schedule(n)) in order, DEPART (partition, to peer)
    after its last bucket.  owner[p]: rank with p's current rows (-1: every
    rank).  Returns (actions, owner after the round)."""
    lib = L.library()
    own = None if owner is None else np.ascontiguousarray(owner, np.int32)
    cnt = np.zeros(1, np.uint64)
    L._check(lib.lgd_round_actions(n, world, rank, r, L._p(own), 0, L._p(cnt), None, None))
    acts = np.zeros(int(cnt[0]), ACTION_DTYPE)
    out = np.zeros(n, np.int32)
    L._check(lib.lgd_round_actions(n, world, rank, r, L._p(own), len(acts), L._p(cnt),
                                   acts.ctypes.data_as(C.c_void_p), L._p(out)))
    return acts, out


def items_as_u64(items: np.ndarray) -> np.ndarray:
    """(count, 8) rows for the oracle: src, dst, g, pool0..2, round, pair."""
    out = np.zeros((len(items), 8), np.uint64)
    out[:, 0] = items["src"]
    out[:, 1] = items["dst"]
    out[:, 2] = items["g"]
    out[:, 3:6] = items["pool"]
    out[:, 6] = items["round"]
    out[:, 7] = items["pair"]
    return out


@dataclass
class Schedule:
    n: int
    world: int
    items: np.ndarray

    @classmethod
    def build(cls, n: int, world: int) -> "Schedule":
        return cls(n, world, round_schedule(n))

    @property
    def num_rounds(self) -> int:
        return int(self.items["round"].max()) + 1 if len(self.items) else 0

    def rank_items(self, r: int, rank: int) -> np.ndarray:
        it = self.items
        sel = (it["round"] == r) & (it["pair"] % self.world == rank)
        return np.ascontiguousarray(it[sel])

    def users(self, r: int) -> dict:
        """partition -> rank that trains on it in round r"""
        it = self.items[self.items["round"] == r]
        out = {}
        for row in it:
            for p in row["pool"]:
                if p != 0xFFFFFFFF:
                    out[int(p)] = int(row["pair"]) % self.world
        return out

    def handoffs(self):
        """Per round: [(partition, from_rank, to_rank)] moves before it runs.
        Every rank starts with an identical copy of every partition."""
        owner = {p: None for p in range(self.n)}
        plan = []
        for r in range(self.num_rounds):
            moves = []
            for p, dst in sorted(self.users(r).items()):
                src = owner[p]
                if src is not None and src != dst:
                    moves.append((p, src, dst))
                owner[p] = dst
            plan.append(moves)
        return plan, owner


class DistComm:
    """torch.distributed communicator (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, dist, device):
        self.dist = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device

    def _drain(self, t=None):
        # the trainer runs on its own stream: finish what torch queued first
        dev = getattr(t, "device", None) if t is not None else self.device
        if str(dev).startswith("cuda"):
            import torch
            torch.cuda.current_stream(dev).synchronize()

    def all_reduce_sum(self, t, drain=True):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        if drain:
            self._drain(t)

    @property
    def stream_ordered(self) -> bool:
        """NCCL on GPUs: the lock-step relation sums can run in stream order
        (Trainer.stream_ordered) instead of draining the host per batch."""
        return str(self.device).startswith("cuda")

    def all_reduce_max_int(self, v: int) -> int:
        import torch
        t = torch.tensor([v], dtype=torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return int(t.item())

    def exchange(self, moves, views):
        """moves: [(p, src, dst)]; views(p) -> list of tensors of partition p"""
        ops = []
        for p, src, dst in moves:
            if self.rank == src:
                ops += [self.dist.P2POp(self.dist.isend, t, dst) for t in views(p)]
            elif self.rank == dst:
                ops += [self.dist.P2POp(self.dist.irecv, t, src) for t in views(p)]
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
            self._drain()


def lock_step(trainer, comm, steps: int, rel_buf):
    """`steps` lock-step batches: this rank's batch, the sum of every rank's
    dense relation gradient, one identical relation Adagrad step.  Over NCCL
    the three run in the trainer's stream order (no host round trip per
    batch: the host only queues work); otherwise each call returns drained."""
    if getattr(comm, "stream_ordered", False) and hasattr(trainer, "stream_ordered"):
        with trainer.stream_ordered():
            for s in range(steps):
                trainer.round_step(s, rel_buf)
                comm.all_reduce_sum(rel_buf, drain=False)
                trainer.round_apply(rel_buf)
        return
    for s in range(steps):
        trainer.round_step(s, rel_buf)
        comm.all_reduce_sum(rel_buf)
        trainer.round_apply(rel_buf)


def run_epoch_actions(trainer, n: int, epoch: int, comm, rel_buf=None, owner=None):
    """One epoch on this rank driven by the C++ runner's plan
    (lgd_round_actions): each round's TRAIN buckets (lock step for typed
    models), then the partitions that DEPART go to their next holder and the
    next round's ARRIVE partitions come in -- the hand-offs lgd_train_round
    does as NVLink pulls, here over the communicator (gloo in the CPU tests).
    Returns (totals, owner after the epoch)."""
    items = round_schedule(n)
    rounds = int(items["round"].max()) + 1 if len(items) else 0
    own = np.full(n, -1, np.int32) if owner is None else np.asarray(owner, np.int32)
    totals = {"loss_sum": 0.0, "edges_trained": 0, "batches": 0, "device_ms": 0.0}
    for r in range(rounds):
        acts, own_after = round_actions(n, comm.world, comm.rank, r, own)
        mine = items[acts["item"][acts["kind"] == TRAIN]]
        if not trainer.typed:
            res = trainer.train_items(epoch, mine)
        else:
            nb = trainer.round_begin(epoch, mine)
            lock_step(trainer, comm, comm.all_reduce_max_int(nb), rel_buf)
            res = trainer.round_end()
        for key in totals:
            totals[key] += getattr(res, key) if hasattr(res, key) else res[key]
        # hand-offs for the next round: my departures, my next arrivals
        moves = [(int(a["part"]), comm.rank, int(a["peer"])) for a in acts if a["kind"] == DEPART]
        if r + 1 < rounds:
            nxt, _ = round_actions(n, comm.world, comm.rank, r + 1, own_after)
            moves += [(int(a["part"]), int(a["peer"]), comm.rank) for a in nxt
                      if a["kind"] == ARRIVE]
        else:
            moves = []  # the epoch's last holders keep their rows (gather_owned)
        comm.exchange(sorted(set(moves)), trainer.partition_views)
        own = own_after
    return totals, own


def gather_owned(trainer, owner, comm):
    """Move every partition from the rank holding its rows to rank 0."""
    moves = [(p, int(o), 0) for p, o in enumerate(owner) if o not in (-1, 0)]
    comm.exchange(moves, trainer.partition_views)


class NativeRounds:
    """The C++ partition-round runner (rounds.cu) on one rank:
    lgd_comm_init(rank, world) -- NCCL for world > 1 -- then lgd_train_round
    per round: the rank's buckets, the hand-offs of the next round's
    partitions as NVLink pulls on a side stream, lock-step NCCL relation
    sums for typed models."""

    def __init__(self, trainer, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        self.trainer, self.rank, self.world = trainer, rank, world
        buf = None
        if world > 1 or nccl_id is not None:  # world 1 with an id: one-rank NCCL communicators
            buf = C.create_string_buffer(bytes(nccl_id), 128)
        L._check(L.library().lgd_comm_init(trainer._h, buf, rank, world))
        cnt = np.zeros(1, np.uint32)
        L._check(L.library().lgd_round_count(trainer._h, L._p(cnt)))
        self.num_rounds = int(cnt[0])

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        L._check(L.library().lgd_comm_unique_id(buf))
        return buf.raw

    def run(self, epoch: int, r: int):
        """-> (EpochResult of this rank's buckets, hand-off ms, hand-off bytes)"""
        res = L._EpochResult()
        ms = np.zeros(1, np.float64)
        nbytes = np.zeros(1, np.uint64)
        L._check(L.library().lgd_train_round(self.trainer._h, epoch, r, C.byref(res), L._p(ms),
                                             L._p(nbytes)))
        return L._result(res), float(ms[0]), int(nbytes[0])


def init_local(trainers):
    """Virtual ranks in one process (lgd_comm_init_local): trainers[q] is rank q."""
    arr = (C.c_void_p * len(trainers))(*[t._h.value for t in trainers])
    L._check(L.library().lgd_comm_init_local(arr, len(trainers)))


def run_round_local(trainers, epoch: int, r: int):
    """One round of virtual ranks: every rank's round queued, then every
    rank's hand-offs, then every rank's results."""
    lib = L.library()
    for t in trainers:
        L._check(lib.lgd_round_enqueue(t._h, epoch, r))
    for t in trainers:
        L._check(lib.lgd_round_handoff(t._h))
    out = []
    for t in trainers:
        res = L._EpochResult()
        ms = np.zeros(1, np.float64)
        nbytes = np.zeros(1, np.uint64)
        L._check(lib.lgd_round_collect(t._h, C.byref(res), L._p(ms), L._p(nbytes)))
        out.append((L._result(res), float(ms[0]), int(nbytes[0])))
    return out


def run_epoch_distributed(trainer, sched: Schedule, epoch: int, comm, rel_buf=None):
    """One epoch of the round schedule on this rank.  `trainer` provides
    train_items / round_begin / round_step / round_apply / round_end /
    partition_views; `rel_buf` is a [R x (d+1)] f64 tensor on the comm device
    (typed models).  Returns this rank's summed EpochResult fields."""
    plan, _ = sched.handoffs()
    totals = {"loss_sum": 0.0, "edges_trained": 0, "batches": 0, "device_ms": 0.0}
    for r in range(sched.num_rounds):
        comm.exchange(plan[r], trainer.partition_views)
        mine = sched.rank_items(r, comm.rank)
        if not trainer.typed:
            res = trainer.train_items(epoch, mine)
        else:
            nb = trainer.round_begin(epoch, mine)
            lock_step(trainer, comm, comm.all_reduce_max_int(nb), rel_buf)
            res = trainer.round_end()
        for key in totals:
            totals[key] += getattr(res, key) if hasattr(res, key) else res[key]
    return totals


def gather_final(trainer, sched: Schedule, comm):
    """Move every partition from its final owner to rank 0."""
    _, owner = sched.handoffs()
    moves = [(p, o, 0) for p, o in sorted(owner.items()) if o not in (None, 0)]
    comm.exchange(moves, trainer.partition_views)


def run_epoch_virtual(trainers, sched: Schedule, epoch: int, copy_partition, rel_bufs=None,
                      sum_into=None, ordered=False):
    """All ranks of the schedule in one process (one trainer per rank, e.g.
    several contexts on one GPU): the 1-GPU parity harness.  ordered=True runs
    the lock-step batches in stream order, the way lock_step does over NCCL:
    the sum waits on every trainer's stream through events, every trainer's
    stream waits on the sum, and the host never drains in between."""
    plan, owner = sched.handoffs()
    world = len(trainers)
    typed = trainers[0].typed

    def drain():  # torch work on the trainers' memory (copies, sums) before they run
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()

    for r in range(sched.num_rounds):
        for p, src, dst in plan[r]:
            copy_partition(trainers[dst], trainers[src], p)
        drain()
        mines = [sched.rank_items(r, q) for q in range(world)]
        if not typed:
            for q in range(world):
                trainers[q].train_items(epoch, mines[q])
            continue
        nbs = [trainers[q].round_begin(epoch, mines[q]) for q in range(world)]
        steps = max(nbs) if nbs else 0
        if ordered:
            _lock_step_virtual_ordered(trainers, steps, rel_bufs, sum_into)
        else:
            for s in range(steps):
                for q in range(world):
                    trainers[q].round_step(s, rel_bufs[q])
                total = sum_into(rel_bufs)
                for q in range(world):
                    trainers[q].round_apply(total)
        for q in range(world):
            trainers[q].round_end()
    for p, o in sorted(owner.items()):
        if o not in (None, 0):
            copy_partition(trainers[0], trainers[o], p)
    drain()


def _lock_step_virtual_ordered(trainers, steps, rel_bufs, sum_into):
    import torch
    streams = [t.cuda_stream() for t in trainers]
    side = torch.cuda.Stream()  # plays NCCL's internal stream
    for t in trainers:
        t.set_stream_ordered(True)
    try:
        for s in range(steps):
            for t, b in zip(trainers, rel_bufs):
                t.round_step(s, b)
            for st in streams:
                side.wait_stream(st)
            with torch.cuda.stream(side):
                total = sum_into(rel_bufs)
            for t, st in zip(trainers, streams):
                st.wait_stream(side)
                total.record_stream(st)
                t.round_apply(total)
    finally:
        for t in trainers:
            t.set_stream_ordered(False)
        for st in streams:
            st.synchronize()


class RoundCursor:
    """Walks the schedule round after round (wrapping into the next epoch)
    and keeps partition ownership across rounds and epochs; every rank starts
    with an identical copy of every partition."""

    def __init__(self, sched: Schedule):
        self.sched = sched
        self.owner = {p: None for p in range(sched.n)}
        self.step = 0

    def next(self):
        """-> (epoch, round, moves) for the next round; ownership advances."""
        r = self.step % self.sched.num_rounds
        epoch = self.step // self.sched.num_rounds
        moves = []
        for p, dst in sorted(self.sched.users(r).items()):
            src = self.owner[p]
            if src is not None and src != dst:
                moves.append((p, src, dst))
            self.owner[p] = dst
        self.step += 1
        return epoch, r, moves


def run_round(trainer, sched: Schedule, epoch: int, r: int, moves, comm, rel_buf=None):
    """One round on this rank: hand-offs, then this rank's buckets (lock-step
    relation sums for typed models).  Returns the trainer's EpochResult."""
    comm.exchange(moves, trainer.partition_views)
    mine = sched.rank_items(r, comm.rank)
    if not trainer.typed:
        return trainer.train_items(epoch, mine)
    nb = trainer.round_begin(epoch, mine)
    lock_step(trainer, comm, comm.all_reduce_max_int(nb), rel_buf)
    return trainer.round_end()
