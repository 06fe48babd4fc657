"""The multi-GPU partition-round runner on CPU: world_size 2 and 3 over gloo,
each rank a trainer backed by the oracle's C arithmetic, driven by the C++
runner's own plan (lgd_round_actions: each rank's buckets per round, the
partitions that depart and arrive, ownership across rounds), with the
hand-offs (send/recv) and lock-step relation sums (all-reduce) over gloo.
The gathered tables must equal the serialised restatement of the same
schedule (oracle run_rounds)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401  (sys.path)

KIND_CASES = ["dot", "distmult", "complex"]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def make_problem(kind):
    rng = np.random.default_rng(3)
    V, R, d, Ecnt, n = 300, 4, 8, 4000, 5
    rels = rng.integers(0, R, Ecnt) if kind != "dot" else np.full(Ecnt, 0xFFFFFFFF)
    edges = np.stack([rng.integers(0, V, Ecnt), rels, rng.integers(0, V, Ecnt)],
                     1).astype(np.uint32)
    return dict(V=V, R=R if kind != "dot" else 0, d=d, edges=edges, n=n, k=3, batch=256, seed=11)


class OracleTrainer:
    """CPU stand-in for lgd.Trainer with the same round-runner interface."""

    def __init__(self, kind, prob, oracle):
        self.kind, self.p, self.o = kind, prob, oracle
        self.typed = kind != "dot"
        V, R, d, n = prob["V"], prob["R"], prob["d"], prob["n"]
        self.E, self.S, rE, rS = oracle.store_init(n, V, d, max(R, 1), 42)
        self.relE, self.relS = (rE, rS) if self.typed else (None, None)
        self.stride, self.offsets, self.order = oracle.partition_plan(prob["edges"], V, n)

    def partition_views(self, p):
        a = self.stride * p
        b = min(self.stride * (p + 1), self.p["V"])
        return [torch.from_numpy(self.E[a:b].reshape(-1)), torch.from_numpy(self.S[a:b].reshape(-1))]

    def _prepare(self, epoch, it):
        n, V = self.p["n"], self.p["V"]
        b = int(it["src"]) * n + int(it["dst"])
        off, m = int(self.offsets[b]), int(self.offsets[b + 1] - self.offsets[b])
        if m == 0:
            return None
        edges = self.p["edges"][self.order[off:off + m]]
        seed = self.o.derive_seed(self.p["seed"], 0x62756B74, epoch, int(it["g"]))
        perm, used = self.o.shuffle_perm(seed, m)
        edges = np.ascontiguousarray(edges[perm])
        parts = sorted(int(q) for q in it["pool"] if q != 0xFFFFFFFF)
        first = [self.stride * q for q in parts]
        count = [min(self.stride * (q + 1), V) - self.stride * q for q in parts]
        negs = self.o.sample_negatives(first, count, self.p["k"], m, seed, skip=used)
        return edges, negs

    def _batches(self, epoch, items):
        out = []
        for it in items:
            prep = self._prepare(epoch, it)
            if prep is None:
                continue
            edges, negs = prep
            k, B = self.p["k"], self.p["batch"]
            for o in range(0, len(edges), B):
                out.append((edges[o:o + B], negs[o * k:(o + B) * k]))
        return out

    def train_items(self, epoch, items):
        loss, cnt = 0.0, 0
        for e, ng in self._batches(epoch, items):
            loss += self.o.batch(self.kind, self.E, self.S, self.relE, self.relS, e, ng,
                                 self.p["k"])["loss"]
            cnt += len(e)
        return {"loss_sum": loss, "edges_trained": cnt, "batches": 0, "device_ms": 0.0}

    def round_begin(self, epoch, items):
        self._queue = self._batches(epoch, items)
        self._acc = {"loss_sum": 0.0, "edges_trained": 0, "batches": 0, "device_ms": 0.0}
        return len(self._queue)

    def round_step(self, s, buf):
        buf.zero_()
        if s < len(self._queue):
            e, ng = self._queue[s]
            loss, dense = self.o.batch_nodes_only(self.kind, self.E, self.S, self.relE, self.relS,
                                                  e, ng, self.p["k"])
            buf.copy_(torch.from_numpy(dense))
            self._acc["loss_sum"] += loss
            self._acc["edges_trained"] += len(e)

    def round_apply(self, summed):
        self.o.adagrad_touched(self.relE, self.relS, summed.numpy())

    def round_end(self):
        return self._acc


def _worker(rank, world, port, kind, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_2505_09258_b200 import multigpu as mg
    prob = make_problem(kind)
    tr = OracleTrainer(kind, prob, Oracle("restatement"))
    comm = mg.DistComm(dist, "cpu")
    rel_buf = torch.zeros((max(prob["R"], 1), prob["d"] + 1), dtype=torch.float64)
    # driven by the C++ runner's plan (lgd_round_actions): buckets per rank and
    # round, departures and arrivals, ownership across rounds
    tot, owner = mg.run_epoch_actions(tr, prob["n"], 0, comm, rel_buf if tr.typed else None)
    mg.gather_owned(tr, owner, comm)
    loss = torch.tensor([tot["loss_sum"]], dtype=torch.float64)
    dist.all_reduce(loss)
    if rank == 0:
        np.savez(out_path, E=tr.E, S=tr.S, relE=tr.relE if tr.typed else np.zeros(1),
                 loss=loss.numpy())
    dist.destroy_process_group()


def _schedule(n):
    """The schedule without a CUDA library load (host planner via ctypes)."""
    from paper_2505_09258_b200 import multigpu as mg
    return mg.round_schedule(n)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", KIND_CASES)
def test_round_runner_matches_serialised_restatement(tmp_path, oracle, kind, world):
    out = str(tmp_path / "final.npz")
    mp.start_processes(_worker, args=(world, free_port(), kind, out), nprocs=world,
                       start_method="spawn", join=True)
    got = np.load(out)
    from paper_2505_09258_b200 import multigpu as mg
    prob = make_problem(kind)
    E, S, rE, rS = oracle.store_init(prob["n"], prob["V"], prob["d"], max(prob["R"], 1), 42)
    items = mg.items_as_u64(_schedule(prob["n"]))
    want = oracle.run_rounds(prob["edges"], prob["V"], prob["R"], prob["n"], items, world, kind,
                             E, S, rE if kind != "dot" else None, rS if kind != "dot" else None,
                             dim=prob["d"], batch_size=prob["batch"], k=prob["k"],
                             seed=prob["seed"])
    assert want["edges_trained"] == len(prob["edges"])
    np.testing.assert_allclose(got["loss"][0], want["loss_sum"], rtol=1e-12)
    if world == 2 or kind == "dot":  # two-term sums are order-free: bit-exact
        assert np.array_equal(got["E"], E) and np.array_equal(got["S"], S)
    else:  # three ranks: the all-reduce may associate the relation sums differently
        np.testing.assert_allclose(got["E"], E, rtol=1e-5, atol=1e-7)
    if kind != "dot":
        np.testing.assert_allclose(got["relE"], rE, rtol=1e-5, atol=1e-7)


def test_schedule_covers_every_bucket_once():
    from paper_2505_09258_b200 import multigpu as mg
    for n in (1, 2, 3, 4, 5, 8, 16, 32):
        it = mg.round_schedule(n)
        buckets = sorted((int(a), int(b)) for a, b in zip(it["src"], it["dst"]))
        assert buckets == [(a, b) for a in range(n) for b in range(n)]
        assert np.array_equal(it["g"], np.arange(len(it)))
        for row in it:  # both endpoints are in the pool
            pool = set(int(q) for q in row["pool"] if q != 0xFFFFFFFF)
            assert {int(row["src"]), int(row["dst"])} <= pool
        for r in np.unique(it["round"]):  # pairs of a round are disjoint
            rows = it[it["round"] == r]
            used = {}
            for row in rows:
                for q in row["pool"]:
                    if q != 0xFFFFFFFF:
                        assert used.setdefault(int(q), int(row["pair"])) == int(row["pair"])


@pytest.mark.parametrize("n", [4, 5, 16, 32])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_round_actions_partition_the_schedule(n, world):
    """lgd_round_actions: every bucket of a round is trained by exactly one
    rank (pair j on rank j % world, in global order); a partition arrives at
    a rank from the rank that held it last, departs to the rank that uses it
    next, and nobody trains a partition it does not hold."""
    from paper_2505_09258_b200 import multigpu as mg
    items = mg.round_schedule(n)
    rounds = int(items["round"].max()) + 1
    owner = np.full(n, -1, np.int32)
    for r in range(rounds):
        got, after = [], None
        for q in range(world):
            acts, own_q = mg.round_actions(n, world, q, r, owner)
            after = own_q if after is None else after
            assert np.array_equal(own_q, after)
            tr = acts["item"][acts["kind"] == mg.TRAIN]
            assert np.all(np.diff(tr.astype(np.int64)) > 0)  # global order
            for i in tr:
                row = items[i]
                assert row["round"] == r and row["pair"] % world == q
                held = {int(p) for p in row["pool"] if p != 0xFFFFFFFF}
                for p in held:  # the rank holds the pool after its arrivals
                    assert after[p] == q
            got += list(tr)
            for a in acts[acts["kind"] == mg.ARRIVE]:
                assert owner[a["part"]] == a["peer"] != q
            for a in acts[acts["kind"] == mg.DEPART]:
                nxt = (r + 1) % rounds
                users = {int(p): int(row["pair"]) % world for row in items[items["round"] == nxt]
                         for p in row["pool"] if p != 0xFFFFFFFF}
                assert users[int(a["part"])] == a["peer"] != q
        assert sorted(got) == list(np.flatnonzero(items["round"] == r))
        owner = after
