"""The C++ partition-round runner (rounds.cu) on one B200 (-m gpu).

* world 1 (lgd_comm_init, no NCCL): an epoch of rounds through
  lgd_train_round equals the serialised restatement (oracle run_rounds);
* virtual ranks (lgd_comm_init_local: one context per rank on the same GPU,
  untyped model): every round's hand-offs run as the runner's peer pulls on
  its side stream, ordered by the ready / arrived events; each partition's
  final rows, read from the rank that holds them, equal the restatement bit
  for bit.  (NCCL lock-step across processes needs one GPU per rank: covered
  by the gloo tests of the same plan, tests/test_multigpu_cpu.py.)
"""
import numpy as np
import pytest

import paper_2505_09258_b200 as lgd
from paper_2505_09258_b200 import multigpu as mg

pytestmark = pytest.mark.gpu
ALL_KINDS = ["dot", "distmult", "complex", "transe"]


def problem(kind, V=3000, Ecnt=60000, n=6, seed=3):
    rng = np.random.default_rng(seed)
    R = 0 if kind == "dot" else 5
    rels = rng.integers(0, R, Ecnt) if R else np.full(Ecnt, 0xFFFFFFFF)
    edges = np.stack([rng.integers(0, V, Ecnt), rels, rng.integers(0, V, Ecnt)],
                     1).astype(np.uint32)
    return dict(V=V, R=R, d=16, edges=edges, n=n, k=4, batch=1500, seed=11)


def trainer(kind, p):
    opts = lgd.TrainOptions(batch_size=p["batch"], negatives=p["k"], seed=p["seed"])
    t = lgd.Trainer(lgd.ScoreModel(kind, p["d"]), opts)
    t.set_graph(p["edges"], p["V"], p["R"])
    t.make_partition_plan(p["n"])
    t.init_store(42)
    return t


def restatement(oracle, kind, p, world):
    E, S, rE, rS = oracle.store_init(p["n"], p["V"], p["d"], max(p["R"], 1), 42)
    items = mg.items_as_u64(mg.round_schedule(p["n"]))
    want = oracle.run_rounds(p["edges"], p["V"], p["R"], p["n"], items, world, kind, E, S,
                             rE if p["R"] else None, rS if p["R"] else None, dim=p["d"],
                             batch_size=p["batch"], k=p["k"], seed=p["seed"])
    return want, E, S, rE


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_train_round_world1_matches_restatement(oracle, kind):
    p = problem(kind)
    t = trainer(kind, p)
    runner = mg.NativeRounds(t, 0, 1)
    loss = edges = 0
    for r in range(runner.num_rounds):
        res, ms, nbytes = runner.run(0, r)
        loss += res.loss_sum
        edges += res.edges_trained
        assert nbytes == 0  # one rank holds every partition
    want, E, S, rE = restatement(oracle, kind, p, 1)
    assert edges == want["edges_trained"] == len(p["edges"])
    assert loss == pytest.approx(want["loss_sum"], rel=1e-12)
    Eg, Sg = t.tables()
    assert np.mean(Eg == E) >= 0.99 and np.linalg.norm(Eg - E) <= 1e-7 * np.linalg.norm(E)
    assert np.mean(Sg == S) >= 0.99
    if p["R"]:
        rEg, _ = t.get_relations()
        assert np.mean(rEg == rE) >= 0.99
    t.close()


@pytest.mark.parametrize("kind", ["dot", "distmult", "complex"])
def test_one_rank_nccl_communicators_match_local_runner(kind):
    """lgd_comm_init with an NCCL id at world 1 builds the multi-process
    machinery for one rank -- libnccl loaded at run time, data + control
    communicators (ncclCommInitRank, ncclCommSplit), the IPC table / event
    handles gathered with ncclAllGather -- and, for typed models, runs the
    lock-step batches with the per-batch ncclAllReduce of the relation
    gradients.  The epoch of rounds equals the local runner's (no NCCL): bit
    for bit for Dot, within the rounds tolerance for typed models (the
    relation step runs as the lock-step kernel instead of the side-stream
    pass)."""
    p = problem(kind)
    got = []
    for nccl in (True, False):
        t = trainer(kind, p)
        runner = mg.NativeRounds(t, 0, 1, nccl_id=mg.NativeRounds.unique_id() if nccl else None)
        loss = 0.0
        for r in range(runner.num_rounds):
            res, ms, nbytes = runner.run(0, r)
            loss += res.loss_sum
        got.append((loss, t.tables()))
        t.close()
    (la, (Ea, Sa)), (lb, (Eb, Sb)) = got
    if kind == "dot":
        assert la == lb
        assert np.array_equal(Ea, Eb) and np.array_equal(Sa, Sb)
    else:
        assert la == pytest.approx(lb, rel=1e-12)
        assert np.mean(Ea == Eb) >= 0.99 and np.linalg.norm(Ea - Eb) <= 1e-7 * np.linalg.norm(Eb)
        assert np.mean(Sa == Sb) >= 0.99


@pytest.mark.parametrize("world", [2, 3])
def test_virtual_ranks_pull_partitions_between_rounds(oracle, world):
    p = problem("dot", n=7)
    ts = [trainer("dot", p) for _ in range(world)]
    mg.init_local(ts)
    owner = np.full(p["n"], -1, np.int32)
    loss = edges = moved = 0
    rounds = int(mg.round_schedule(p["n"])["round"].max()) + 1
    for r in range(rounds):
        for res, ms, nbytes in mg.run_round_local(ts, 0, r):
            loss += res.loss_sum
            edges += res.edges_trained
            moved += nbytes
        owner = mg.round_actions(p["n"], world, 0, r, owner)[1]
    assert moved > 0
    want, E, S, _ = restatement(oracle, "dot", p, world)
    assert edges == want["edges_trained"]
    assert loss == pytest.approx(want["loss_sum"], rel=1e-12)
    stride = -(-p["V"] // p["n"])
    for q in range(p["n"]):
        holder = ts[int(owner[q])] if owner[q] >= 0 else ts[0]
        blob = holder.store_partition(q).reshape(2, -1, p["d"])
        sl = slice(stride * q, min(stride * (q + 1), p["V"]))
        assert np.array_equal(blob[0], E[sl]), q
        assert np.array_equal(blob[1], S[sl]), q
    for t in ts:
        t.close()
