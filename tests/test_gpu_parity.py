"""CUDA path vs the oracle (C restatement of the reference) and the golden
vectors generated from the reference library.  Runs on a B200 (-m gpu).

Tolerances (stated here):
  * indices -- shuffled order, negative ids, partition plan, eval candidates,
    unique-row counts: bit-exact;
  * store init: bit-exact (integer-seeded f32);
  * per-batch loss / epoch loss_sum: |rel| <= 1e-12 (the kernels compute in
    FP64 like the reference; only the dot-product summation order and
    exp/log ulps differ);
  * gradients: |rel| <= 1e-10 per row norm;
  * embeddings / Adagrad state after training: relative Frobenius <= 1e-7
    per partition and >= 99% of elements bit-identical.
"""
import numpy as np
import pytest
from conftest import golden

import paper_2505_09258_b200 as lgd

pytestmark = pytest.mark.gpu
KINDS = ["dot", "distmult", "complex"]
# TransE is not in the reference: it is checked against the restatement only
# (oracle/legend_oracle.c defines it; "parity unpinned" in DESIGN.md)
ALL_KINDS = KINDS + ["transe"]


def frob(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def assert_tables_close(got, want, what):
    assert got.shape == want.shape, what
    assert frob(got, want) <= 1e-7, (what, frob(got, want))
    same = np.mean(got == want)
    assert same >= 0.99, (what, same)


def make_trainer(kind, d, V, R, edges, n, k=16, batch=100000, seed=42, shuffle=True, lr=0.1):
    opts = lgd.TrainOptions(learning_rate=lr, batch_size=batch, negatives=k, shuffle=shuffle,
                            seed=seed)
    t = lgd.Trainer(lgd.ScoreModel(kind, d), opts)
    t.set_graph(edges, V, R)
    t.make_partition_plan(n)
    return t


# ------------------------------------------------------------------ K2 / K1
def test_rng_below_rejection_path_matches_golden():
    g = golden("rng")
    vals, used = lgd.rng_below(int(g["reject_seed"]), 2**63 + 1, 5000, skip=int(g["reject_skip"]))
    assert np.array_equal(vals, g["reject_vals"])
    assert used == int(g["reject_used"])


@pytest.mark.parametrize("bound", [1, 2, 7, 1000, 7_800_000, 2**32 - 1, 2**40 + 3])
def test_rng_below_matches_oracle(oracle, bound):
    for count, skip in ((1, 0), (1000, 3), (300_000, 12345)):
        vals, used = lgd.rng_below(77, bound, count, skip=skip)
        want, wused = oracle.rng_below(77, np.full(count, bound, np.uint64), skip=skip)
        assert np.array_equal(vals, want)
        assert used == wused


def test_sample_negatives_match_golden():
    g = golden("sampler")
    s2, _ = lgd.sample_negatives(g["first2"], g["count2"], 4, 2500, 4242)
    assert np.array_equal(s2, g["s2"])
    s3, used = lgd.sample_negatives(g["first3"], g["count3"], 16, 5000, 99, skip=12345)
    assert np.array_equal(s3, g["s3"])
    assert used == 16 * 5000


def test_sample_negatives_large_matches_oracle(oracle):
    # a Twitter-shaped pool (3 x 2.6M resident rows), one bucket's worth of draws
    first = [2_600_000 * 2, 2_600_000 * 7, 2_600_000 * 11]
    count = [2_600_000, 2_600_000, 2_600_000]
    got, used = lgd.sample_negatives(first, count, 16, 1_000_000, 123456789, skip=5_099_999)
    want = oracle.sample_negatives(first, count, 16, 1_000_000, 123456789, skip=5_099_999)
    assert used == 16_000_000
    assert np.array_equal(got, want)


@pytest.mark.parametrize("m", [0, 1, 2, 3, 10, 1000, 65_537, 1_000_000])
def test_shuffle_permutation_matches_oracle(oracle, m):
    seed = 0x1234567 + m
    got, used = lgd.shuffle_permutation(seed, m)
    want, wused = oracle.shuffle_perm(seed, m)
    assert np.array_equal(got, want)
    assert used == wused


def test_shuffle_permutation_twitter_bucket(oracle):
    m = 5_100_000  # mean Twitter bucket (1.3B edges / 256 buckets)
    got, used = lgd.shuffle_permutation(987654321, m)
    want, _ = oracle.shuffle_perm(987654321, m)
    assert np.array_equal(got, want)
    assert np.array_equal(np.sort(got), np.arange(m, dtype=np.uint32))


# ----------------------------------------------------- loader / store init
def test_partition_plan_matches_golden():
    g = golden("partition")
    t = make_trainer("dot", 4, int(g["V"]), 3, g["edges"], int(g["n"]))
    offsets, order = t.make_partition_plan(int(g["n"]), want_edge_order=True)
    assert np.array_equal(offsets, g["offsets"])
    assert np.array_equal(order, g["edge_order"])


def test_store_init_matches_golden():
    g = golden("store")
    V, R, n, d = int(g["V"]), int(g["R"]), int(g["n"]), int(g["dim"])
    edges = np.array([[0, 0, 1]], np.uint32)
    t = make_trainer("distmult", d, V, R, edges, n)
    t.init_store(int(g["seed"]))
    E, S = t.tables()
    rE, rS = t.get_relations()
    assert np.array_equal(E, g["E"]) and not S.any()
    assert np.array_equal(rE, g["relE"]) and not rS.any()


# ------------------------------------------------------ K3 / K4 one batch
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("d", [6, 12])
def test_batch_matches_golden(kind, d):
    g = golden(f"batch_{kind}_d{d}")
    V, R, k = g["E0"].shape[0], g["rE0"].shape[0], int(g["k"])
    t = make_trainer(kind, d, V, R if kind != "dot" else 0, g["edges"], 1, k=k)
    t.load_tables(g["E0"], g["S0"])
    if kind != "dot":
        t.set_relations(g["rE0"], g["rS0"])
    gr = t.batch_gradients(g["edges"], g["negs"])
    assert gr["loss"] == pytest.approx(float(g["loss"]), rel=1e-12)
    assert np.array_equal(gr["node_ids"], g["node_ids"])
    np.testing.assert_allclose(gr["node_grads"], g["node_grads"], rtol=1e-10, atol=1e-14)
    if kind != "dot":
        assert np.array_equal(gr["rel_ids"], g["rel_ids"])
        np.testing.assert_allclose(gr["rel_grads"], g["rel_grads"], rtol=1e-10, atol=1e-14)
    res = t.train_batch(g["edges"], g["negs"])
    assert res["loss"] == pytest.approx(float(g["loss"]), rel=1e-12)
    assert res["nodes"] == len(g["node_ids"])
    E, S = t.tables()
    assert_tables_close(E, g["E1"], "E")
    assert_tables_close(S, g["S1"], "S")
    if kind != "dot":
        rE, rS = t.get_relations()
        assert_tables_close(rE, g["rE1"], "relE")
        assert_tables_close(rS, g["rS1"], "relS")


@pytest.mark.parametrize("kind", ALL_KINDS)
@pytest.mark.parametrize("d,k,P,V", [(100, 16, 3000, 5000), (64, 5, 777, 5000),
                                     (128, 40, 500, 5000), (32, 1, 64, 5000),
                                     (100, 16, 3000, 64), (100, 16, 3000, 2000),
                                     (200, 8, 1000, 3000), (36, 3, 2000, 300)])
def test_batch_matches_oracle_wide(oracle, kind, d, k, P, V):
    """Segment lengths from 1 to ~850 contributions (V=64): chunk-boundary
    crossings, short-segment extension and long (pass-2) segments."""
    rng = np.random.default_rng(d * 1000 + k + V)
    R = 17
    E0 = rng.uniform(-0.05, 0.05, (V, d)).astype(np.float32)
    S0 = rng.uniform(0, 0.01, (V, d)).astype(np.float32)
    rE0 = rng.uniform(-0.05, 0.05, (R, d)).astype(np.float32)
    rS0 = np.zeros((R, d), np.float32)
    rels = rng.integers(0, R, P) if kind != "dot" else np.full(P, 0xFFFFFFFF)
    # a hub node to exercise long segments (chunk-spanning reductions)
    src = np.where(rng.random(P) < 0.3, 17, rng.integers(0, V, P))
    edges = np.stack([src, rels, rng.integers(0, V, P)], 1).astype(np.uint32)
    negs = rng.integers(0, V, P * k).astype(np.uint32)
    t = make_trainer(kind, d, V, R if kind != "dot" else 0, edges, 1, k=k)
    t.load_tables(E0, S0)
    if kind != "dot":
        t.set_relations(rE0, rS0)
    E, S, rE, rS = E0.copy(), S0.copy(), rE0.copy(), rS0.copy()
    want = oracle.batch(kind, E, S, rE if kind != "dot" else None, rS if kind != "dot" else None,
                        edges, negs, k)
    got = t.train_batch(edges, negs)
    assert got["loss"] == pytest.approx(want["loss"], rel=1e-12)
    assert got["nodes"] == want["nodes"] and got["rels"] == want["rels"]
    Eg, Sg = t.tables()
    assert_tables_close(Eg, E, "E")
    assert_tables_close(Sg, S, "S")
    if kind != "dot":
        rEg, rSg = t.get_relations()
        assert_tables_close(rEg, rE, "relE")


# ------------------------------------------------------------ full epochs
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n", [1, 4])
def test_epoch_matches_golden(kind, n):
    g = golden(f"epoch_{kind}_n{n}")
    V, R, d = int(g["V"]), int(g["R"]), int(g["d"])
    t = make_trainer(kind, d, V, R if kind != "dot" else 0, g["edges"], n, k=int(g["k"]),
                     batch=int(g["batch"]), seed=int(g["seed"]))
    t.init_store(int(g["store_seed"]))
    res = t.run_epoch(0)
    assert res.edges_trained == int(g["edges_trained"])
    assert res.buckets_trained == int(g["buckets_trained"])
    assert res.batches == len(g["batch_loss"])
    assert res.unique_nodes == int(g["batch_nodes"].sum())  # bit-exact index work
    assert res.unique_rels == int(g["batch_rels"].sum())
    assert res.loss_sum == pytest.approx(float(g["loss_sum"]), rel=1e-12)
    E, S = t.tables()
    assert_tables_close(E, g["E"], "E")
    assert_tables_close(S, g["S"], "S")
    if kind != "dot":
        rE, rS = t.get_relations()
        assert_tables_close(rE, g["relE"], "relE")
        assert_tables_close(rS, g["relS"], "relS")


@pytest.mark.parametrize("kind", KINDS)
def test_evaluate_matches_golden(kind):
    g = golden(f"eval_{kind}")
    E, rE, test = g["E"], g["relE"], g["test"]
    R = rE.shape[0] if kind != "dot" else 0
    t = make_trainer(kind, E.shape[1], E.shape[0], R, test, 1)
    t.load_tables(E, np.zeros_like(E))
    if R:
        t.set_relations(rE, np.zeros_like(rE))
    mrr, hits = t.evaluate(test, lgd.EvalOptions(hits_k=10, num_candidates=999,
                                                 seed=int(g["seed"])))
    assert mrr == pytest.approx(float(g["mrr"]), rel=1e-12)
    assert hits == pytest.approx(float(g["hits"]), abs=1e-12)


# ------------------------------------------------- TransE vs restatement
@pytest.mark.parametrize("n", [1, 4])
def test_transe_epoch_matches_restatement(oracle, n):
    """Same graphs / plans as the DistMult epoch fixtures, TransE scores."""
    g = golden(f"epoch_distmult_n{n}")
    V, R, d, k, B = int(g["V"]), int(g["R"]), int(g["d"]), int(g["k"]), int(g["batch"])
    t = make_trainer("transe", d, V, R, g["edges"], n, k=k, batch=B, seed=int(g["seed"]))
    t.init_store(int(g["store_seed"]))
    res = t.run_epoch(0)
    E, S, rE, rS = oracle.store_init(n, V, d, R, int(g["store_seed"]))
    plan = dict(states=g["states"], bucket_order=g["bucket_order"],
                state_offsets=g["state_offsets"])
    want = oracle.run_epoch(g["edges"], V, R, n, plan, "transe", E, S, rE, rS, dim=d,
                            batch_size=B, k=k, seed=int(g["seed"]), dumps=True)
    assert res.edges_trained == want["edges_trained"]
    assert res.unique_nodes == int(want["batch_nodes"].sum())
    assert res.loss_sum == pytest.approx(want["loss_sum"], rel=1e-12)
    Eg, Sg = t.tables()
    assert_tables_close(Eg, E, "E")
    assert_tables_close(Sg, S, "S")
    rEg, rSg = t.get_relations()
    assert_tables_close(rEg, rE, "relE")
    assert_tables_close(rSg, rS, "relS")


def test_transe_zero_distance_edges(oracle):
    """u == t exactly (self loops over a zero relation row, and negatives equal
    to the positive): the 1/D coefficients are defined as 0 there."""
    V, R, d, k = 50, 3, 16, 4
    rng = np.random.default_rng(9)
    E0 = rng.uniform(-0.05, 0.05, (V, d)).astype(np.float32)
    rE0 = rng.uniform(-0.05, 0.05, (R, d)).astype(np.float32)
    rE0[0] = 0.0
    P = 400
    src = rng.integers(0, V, P)
    rel = rng.integers(0, R, P)
    dst = np.where(rel == 0, src, rng.integers(0, V, P))
    edges = np.stack([src, rel, dst], 1).astype(np.uint32)
    negs = np.where(rng.random((P, k)) < 0.3, dst[:, None],
                    rng.integers(0, V, (P, k))).astype(np.uint32).reshape(-1)
    t = make_trainer("transe", d, V, R, edges, 1, k=k)
    t.load_tables(E0, np.zeros_like(E0))
    t.set_relations(rE0, np.zeros_like(rE0))
    E, S, rE, rS = E0.copy(), np.zeros_like(E0), rE0.copy(), np.zeros_like(rE0)
    gr = t.batch_gradients(edges, negs)
    want_g = oracle.batch("transe", E.copy(), S.copy(), rE.copy(), rS.copy(), edges, negs, k,
                          apply=False, grads=True)
    assert np.isfinite(gr["node_grads"]).all()
    assert np.array_equal(gr["node_ids"], want_g["node_ids"])
    np.testing.assert_allclose(gr["node_grads"], want_g["node_grads"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(gr["rel_grads"], want_g["rel_grads"], rtol=1e-10, atol=1e-14)
    want = oracle.batch("transe", E, S, rE, rS, edges, negs, k)
    got = t.train_batch(edges, negs)
    assert got["loss"] == pytest.approx(want["loss"], rel=1e-12)
    Eg, Sg = t.tables()
    assert_tables_close(Eg, E, "E")
    assert_tables_close(Sg, S, "S")


def test_transe_evaluate_matches_restatement(oracle):
    g = golden("eval_distmult")
    E, rE, test = g["E"], g["relE"], g["test"]
    t = make_trainer("transe", E.shape[1], E.shape[0], rE.shape[0], test, 1)
    t.load_tables(E, np.zeros_like(E))
    t.set_relations(rE, np.zeros_like(rE))
    mrr, hits = t.evaluate(test, lgd.EvalOptions(hits_k=10, num_candidates=999,
                                                 seed=int(g["seed"])))
    wmrr, whits = oracle.evaluate("transe", E, rE, test, 999, 10, int(g["seed"]))
    assert mrr == pytest.approx(wmrr, rel=1e-12)
    assert hits == pytest.approx(whits, abs=1e-12)


# ------------------------------------------- configs[0]: FB15k-shaped KG
def test_fb15k_shaped_distmult_epoch_matches_oracle(oracle):
    """BASELINE configs[0]: 15k nodes, 1,345 relations, 592k edges, DistMult
    d=100, 1 partition, k=16, P=1e5 -- full epoch vs the restatement."""
    rng = np.random.default_rng(15)
    V, R, Ecnt, d = 15000, 1345, 592_000, 100
    edges = np.stack([rng.integers(0, V, Ecnt), rng.integers(0, R, Ecnt),
                      rng.integers(0, V, Ecnt)], 1).astype(np.uint32)
    t = make_trainer("distmult", d, V, R, edges, 1, k=16, batch=100000, seed=42)
    t.init_store(42)
    res = t.run_epoch(0)
    E, S, rE, rS = oracle.store_init(1, V, d, R, 42)
    from oracle.oracle import single_state_plan
    want = oracle.run_epoch(edges, V, R, 1, single_state_plan(1), "distmult", E, S, rE, rS,
                            dim=d, batch_size=100000, k=16, seed=42, dumps=True)
    assert res.edges_trained == want["edges_trained"] == Ecnt
    assert res.unique_nodes == int(want["batch_nodes"].sum())
    assert res.loss_sum == pytest.approx(want["loss_sum"], rel=1e-12)
    Eg, Sg = t.tables()
    assert_tables_close(Eg, E, "E")
    assert_tables_close(Sg, S, "S")
    rEg, rSg = t.get_relations()
    assert_tables_close(rEg, rE, "relE")
    assert_tables_close(rSg, rS, "relS")


# ------------------------------------------------------- error behaviour
def test_errors_follow_reference_classes():
    edges = np.array([[0, 0, 1], [1, 0, 2]], np.uint32)
    t = make_trainer("distmult", 8, 10, 0, np.array([[0, 0xFFFFFFFF, 1]], np.uint32), 1)
    t.init_store(1)
    with pytest.raises(lgd.InvalidArgument):  # typed model, no relations (pipeline.cpp:228)
        t.run_epoch(0)
    t2 = make_trainer("distmult", 8, 10, 2, edges, 1, k=2)
    t2.init_store(1)
    with pytest.raises(lgd.OutOfRange):  # node not resident (train.cpp:157)
        t2.train_batch(np.array([[0, 0, 99]], np.uint32), np.array([1, 2], np.uint32))
    with pytest.raises(lgd.InvalidArgument):  # missing relation id (train.cpp:209-211)
        t2.train_batch(np.array([[0, 0xFFFFFFFF, 1]], np.uint32), np.array([1, 2], np.uint32))
    with pytest.raises(lgd.InvalidArgument):
        make_trainer("dot", 8, 10, 0, edges, 11)  # n > V (graph.cpp:122)


# ------------------------------------------- multi-GPU round schedule (1 GPU)
@pytest.mark.parametrize("kind", ALL_KINDS)
@pytest.mark.parametrize("world,ordered", [(1, False), (2, False), (3, False), (1, True),
                                           (3, True)])
def test_round_schedule_virtual_ranks_match_restatement(oracle, kind, world, ordered):
    """`world` trainer contexts on one GPU run the partition-round schedule
    exactly as `world` GPUs would (hand-offs as device copies, lock-step
    relation sums); the result must match the serialised restatement.
    ordered: the lock-step batches run in stream order with no host drain
    between a batch, the relation sum and the relation step (lock_step's
    NCCL mode)."""
    import torch
    from paper_2505_09258_b200 import multigpu as mg
    rng = np.random.default_rng(21)
    V, R, d, Ecnt, n, k, B = 500, 5, 12, 8000, 6, 4, 300
    rels = rng.integers(0, R, Ecnt) if kind != "dot" else np.full(Ecnt, 0xFFFFFFFF)
    edges = np.stack([rng.integers(0, V, Ecnt), rels, rng.integers(0, V, Ecnt)],
                     1).astype(np.uint32)
    Rm = R if kind != "dot" else 0
    trainers = [make_trainer(kind, d, V, Rm, edges, n, k=k, batch=B, seed=7) for _ in range(world)]
    for t in trainers:
        t.init_store(42)
    sched = mg.Schedule.build(n, world)

    def copy_partition(dst, src, p):
        for a, b in zip(dst.partition_views(p), src.partition_views(p)):
            a.copy_(b)

    bufs = [torch.zeros((max(Rm, 1), d + 1), dtype=torch.float64, device="cuda")
            for _ in range(world)]

    def sum_into(bs):
        total = bs[0].clone()
        for b in bs[1:]:
            total += b
        return total

    mg.run_epoch_virtual(trainers, sched, 0, copy_partition, bufs, sum_into, ordered=ordered)
    torch.cuda.synchronize()
    E, S = trainers[0].tables()
    E0, S0, rE, rS = oracle.store_init(n, V, d, max(Rm, 1), 42)
    want = oracle.run_rounds(edges, V, Rm, n, mg.items_as_u64(sched.items), world, kind, E0, S0,
                             rE if Rm else None, rS if Rm else None, dim=d, batch_size=B, k=k,
                             seed=7)
    assert want["edges_trained"] == Ecnt
    assert_tables_close(E, E0, "E")
    assert_tables_close(S, S0, "S")
    if Rm:
        rEg, rSg = trainers[0].get_relations()
        assert_tables_close(rEg, rE, "relE")


# ------------------------------------------------ host-streamed bucket input
def test_host_edges_path_matches_device_path():
    """lgd_set_host_edges / train_buckets_from_host stream each bucket H2D; the
    trained tables and losses equal the device-resident path bit for bit."""
    rng = np.random.default_rng(8)
    V, R, d, Ecnt, n = 3000, 6, 32, 60000, 4
    edges = np.stack([rng.integers(0, V, Ecnt), rng.integers(0, R, Ecnt),
                      rng.integers(0, V, Ecnt)], 1).astype(np.uint32)
    a = make_trainer("distmult", d, V, R, edges, n, k=8, batch=4000)
    b = make_trainer("distmult", d, V, R, edges, n, k=8, batch=4000)
    a.init_store(3)
    b.init_store(3)
    ra = a.run_epoch(0)
    host = lgd.PinnedArray((b.num_edges, 3), np.uint32)
    b.bucketed_edges(host.array)
    b.set_host_edges(host.array)
    rb = b.run_epoch(0)
    b.set_host_edges(None)
    host.free()
    assert rb.loss_sum == ra.loss_sum and rb.edges_trained == ra.edges_trained
    assert rb.h2d_bytes == 12 * Ecnt
    Ea, Sa = a.tables()
    Eb, Sb = b.tables()
    assert np.array_equal(Ea, Eb) and np.array_equal(Sa, Sb)
    assert np.array_equal(a.get_relations()[0], b.get_relations()[0])


# --------------------------------------------------- bucket-level presort
@pytest.mark.parametrize("kind", ALL_KINDS)
def test_bucket_presort_matches_per_batch_sort(kind, monkeypatch):
    """The bucket-level contribution sort (one radix sort of (batch, pool
    index) keys per bucket) gives every batch the run its own sort would:
    losses, counts and tables equal the per-batch-sort path bit for bit,
    ragged last batches included."""
    rng = np.random.default_rng(11)
    V, R, d, Ecnt, n = 2500, 5, 16, 50000, 4
    edges = np.stack([rng.integers(0, V, Ecnt), rng.integers(0, R, Ecnt),
                      rng.integers(0, V, Ecnt)], 1).astype(np.uint32)
    R = R if kind != "dot" else 0
    runs = []
    for presort in ("1", "0"):
        monkeypatch.setenv("LGD_PRESORT", presort)
        t = make_trainer(kind, d, V, R, edges, n, k=8, batch=700)
        t.init_store(5)
        res = t.run_epoch(0)
        runs.append((res, t.tables(), t.get_relations() if R else None))
    (ra, (Ea, Sa), rela), (rb, (Eb, Sb), relb) = runs
    assert ra.loss_sum == rb.loss_sum and ra.batches == rb.batches
    assert ra.unique_nodes == rb.unique_nodes and ra.unique_rels == rb.unique_rels
    assert np.array_equal(Ea, Eb) and np.array_equal(Sa, Sb)
    if R:
        assert np.array_equal(rela[0], relb[0]) and np.array_equal(rela[1], relb[1])


# ------------------------------------------- asynchronous partition write-back
@pytest.mark.parametrize("kind", ["distmult", "dot"])
def test_async_store_overlaps_eval_and_orders_before_training(kind):
    """lgd_store_partition_async (the epoch-end writes of pipeline.cpp:173-193):
    the pinned copies see the tables exactly as the epoch left them, an
    evaluate queued behind them runs unchanged, and the next epoch -- which
    rewrites every partition -- is ordered after the copies."""
    g = golden(f"epoch_{kind}_n4")
    V, R, d = int(g["V"]), int(g["R"]), int(g["d"])
    t = make_trainer(kind, d, V, R if kind != "dot" else 0, g["edges"], 4, k=int(g["k"]),
                     batch=int(g["batch"]), seed=int(g["seed"]))
    t.init_store(int(g["store_seed"]))
    t.run_epoch(0)
    want = [t.store_partition(p) for p in range(4)]
    test = np.asarray(g["edges"][:200])
    ev = lgd.EvalOptions(hits_k=10, num_candidates=99, seed=7)
    mrr0, hits0 = t.evaluate(test, ev)
    bufs = [lgd.PinnedArray(w.shape, np.float32) for w in want]
    for p, b in enumerate(bufs):
        b.array[:] = np.nan
        t.store_partition_async(p, b.array)
    mrr1, hits1 = t.evaluate(test, ev)  # read-only: may overlap the copies
    t.run_epoch(1)  # writes the tables: ordered after the copies
    t.wait_stores()
    for p in range(4):
        np.testing.assert_array_equal(bufs[p].array, want[p])
    assert (mrr1, hits1) == (mrr0, hits0)
    assert not np.array_equal(t.store_partition(0), want[0])  # epoch 1 did train
    with pytest.raises(ValueError):
        t.store_partition_async(0, np.zeros(3, np.float32))
    t.close()
    for b in bufs:
        b.free()


# ------------------------------------------- K4 v2: segment-list row updates
def _hub_graph(rng, V, R, E):
    src = rng.integers(0, V, E)
    dst = rng.integers(0, V, E)
    dst[rng.random(E) < 0.25] = 11  # a hub: segments of thousands of contributions
    src[rng.random(E) < 0.10] = 12
    return np.stack([src, rng.integers(0, max(R, 1), E), dst], 1).astype(np.uint32)


@pytest.mark.parametrize("kind", ALL_KINDS)
def test_k4_segment_rows_sum_hubs_in_reference_order(oracle, kind, monkeypatch):
    """K4 v2 (segment_rows, the default: segments of <= 32 contributions summed
    whole in the reference's std::map order, hubs in 32-item chunks added in
    chunk order) and the chunked kernels (LGD_K4=1) both stay within the
    stated tolerance of the restatement, with exact unique-row counts."""
    rng = np.random.default_rng(21)
    V, R, d, Ecnt, n, k, B = 4000, 6, 36 if kind != "complex" else 40, 40000, 4, 8, 3000
    R = R if kind != "dot" else 0
    edges = _hub_graph(rng, V, R, Ecnt)
    if not R:
        edges[:, 1] = 0xFFFFFFFF
    plan = lgd.plan_iteration_order(n).as_dict()
    E0, S0, rE0, rS0 = oracle.store_init(n, V, d, R, 5)
    want = oracle.run_epoch(edges, V, R, n, plan, kind, E0, S0, rE0, rS0, dim=d, batch_size=B,
                            k=k, seed=42, dumps=True)
    same = {}
    for mode in ("2", "1"):
        monkeypatch.setenv("LGD_K4", mode)
        t = make_trainer(kind, d, V, R, edges, n, k=k, batch=B)
        t.init_store(5)
        res = t.run_epoch(0)
        assert res.unique_nodes == int(want["batch_nodes"].sum())
        assert res.loss_sum == pytest.approx(want["loss_sum"], rel=1e-12)
        Eg, Sg = t.tables()
        assert_tables_close(Eg, E0, f"E K4={mode}")
        assert_tables_close(Sg, S0, f"S K4={mode}")
        same[mode] = np.mean(Eg == E0)
        t.close()
    assert min(same.values()) >= 0.99, same


@pytest.mark.parametrize("kind", ["complex", "transe"])
def test_k4_ir1_rows_equal_snapshot_recombination(kind, monkeypatch):
    """ComplEx / TransE: K4 reading K3's FP64 IR1 rows (default) and K4
    recombining the src snapshot with the relation row (LGD_K4_IR1=0) form
    the same expression, so losses, counts and tables are bit-identical."""
    rng = np.random.default_rng(13)
    V, R, d, Ecnt, n = 2500, 5, 16, 50000, 4
    edges = _hub_graph(rng, V, R, Ecnt)
    runs = []
    for ir1 in ("1", "0"):
        monkeypatch.setenv("LGD_K4_IR1", ir1)
        t = make_trainer(kind, d, V, R, edges, n, k=8, batch=700)
        t.init_store(5)
        res = t.run_epoch(0)
        runs.append((res, t.tables(), t.get_relations()))
        t.close()
    (ra, (Ea, Sa), rela), (rb, (Eb, Sb), relb) = runs
    assert ra.loss_sum == rb.loss_sum and ra.unique_nodes == rb.unique_nodes
    assert np.array_equal(Ea, Eb) and np.array_equal(Sa, Sb)
    assert np.array_equal(rela[0], relb[0]) and np.array_equal(rela[1], relb[1])


# ------------------------------------ next-bucket prep on its own stream
@pytest.mark.parametrize("kind,host,shared", [("distmult", False, 0), ("complex", True, 0),
                                               ("dot", False, 0), ("transe", True, 0),
                                               ("distmult", False, 50)])
def test_overlapped_bucket_prep_matches_serial(kind, host, shared, monkeypatch):
    """LGD_OVERLAP_PREP=1 (opt-in): the next bucket's shuffle, sample,
    presort and segment list run on a low-priority stream into the second
    buffer set while the current bucket's batches train.  Two epochs, device
    or host-streamed edges, exact or shared negatives: losses, counts and
    tables equal the serial path (LGD_OVERLAP_PREP=0) bit for bit."""
    rng = np.random.default_rng(17)
    V, R, d, Ecnt, n = 3000, 5, 16, 60000, 4
    edges = _hub_graph(rng, V, R, Ecnt)
    R = R if kind != "dot" else 0
    if not R:
        edges[:, 1] = 0xFFFFFFFF
    runs = []
    for ovl in ("1", "0"):
        monkeypatch.setenv("LGD_OVERLAP_PREP", ovl)
        opts = lgd.TrainOptions(batch_size=900, negatives=8, seed=3, shared_chunk=shared)
        t = lgd.Trainer(lgd.ScoreModel(kind, d), opts)
        t.set_graph(edges, V, R)
        t.make_partition_plan(n)
        t.init_store(5)
        pinned = None
        if host:
            pinned = lgd.PinnedArray((t.num_edges, 3), np.uint32)
            t.bucketed_edges(pinned.array)
            t.set_host_edges(pinned.array)
        res = [t.run_epoch(e) for e in range(2)]
        if host:
            t.set_host_edges(None)
            pinned.free()
        runs.append(([(r.loss_sum, r.batches, r.unique_nodes, r.unique_rels) for r in res],
                     t.tables(), t.get_relations() if R else None))
        t.close()
    (la, (Ea, Sa), rela), (lb, (Eb, Sb), relb) = runs
    assert la == lb
    assert np.array_equal(Ea, Eb) and np.array_equal(Sa, Sb)
    if R:
        assert np.array_equal(rela[0], relb[0]) and np.array_equal(rela[1], relb[1])
