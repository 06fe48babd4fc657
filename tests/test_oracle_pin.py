"""Pin the C restatement (oracle/legend_oracle.c) to the reference: golden
vectors generated from the reference library, the reference's own
known-answer tests (test_train.cpp), and -- where the reference library was
built here -- randomized head-to-head runs.  CPU only."""
import numpy as np
import pytest
from conftest import golden

KINDS = ["dot", "distmult", "complex"]


def test_rng_streams_match_golden(oracle):
    g = golden("rng")
    for args, want in zip(g["derive_in"], g["derive_out"]):
        assert oracle.derive_seed(*[int(a) for a in args]) == int(want)
    assert np.array_equal(oracle.rng_u64(int(g["raw_seed"]), len(g["raw"])), g["raw"])
    vals, used = oracle.rng_below(int(g["below_seed"]), g["below_bounds"])
    assert np.array_equal(vals, g["below_vals"]) and used == int(g["below_used"])
    # bound 2^63+1 rejects about half the raw draws (rng.hpp:43-46)
    vals, used = oracle.rng_below(int(g["reject_seed"]), np.full(5000, 2**63 + 1, np.uint64),
                                  skip=int(g["reject_skip"]))
    assert np.array_equal(vals, g["reject_vals"]) and used == int(g["reject_used"])
    assert used > 5000 + 2000


def test_sampler_matches_golden(oracle):
    g = golden("sampler")
    assert np.array_equal(oracle.sample_negatives(g["first2"], g["count2"], 4, 2500, 4242), g["s2"])
    assert np.array_equal(
        oracle.sample_negatives(g["first3"], g["count3"], 16, 5000, 99, skip=12345), g["s3"])


def test_sampler_uniform_chi_square(oracle):
    # test_train.cpp:231-267: two resident ranges, chi-square vs uniform
    s = oracle.sample_negatives([0, 100], [50, 50], 4, 2500, 4242)
    assert np.all((s < 50) | ((s >= 100) & (s < 150)))
    counts = np.bincount(np.where(s < 50, s, s - 50), minlength=100)
    chi2 = ((counts - 100.0) ** 2 / 100.0).sum()
    assert chi2 < 99 + 4 * np.sqrt(2 * 99)


def test_partition_plan_matches_golden(oracle):
    g = golden("partition")
    stride, off, order = oracle.partition_plan(g["edges"], int(g["V"]), int(g["n"]))
    assert stride == int(g["stride"])
    assert np.array_equal(off, g["offsets"]) and np.array_equal(order, g["edge_order"])


def test_store_init_matches_golden(oracle):
    g = golden("store")
    E, S, rE, rS = oracle.store_init(int(g["n"]), int(g["V"]), int(g["dim"]), int(g["R"]),
                                     int(g["seed"]))
    assert np.array_equal(E, g["E"]) and np.array_equal(rE, g["relE"])
    assert not S.any() and not rS.any()
    bound = 0.5 / np.sqrt(int(g["dim"]))
    assert np.abs(E).max() <= bound


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("d", [6, 12])
def test_batch_matches_golden_bitwise(oracle, kind, d):
    g = golden(f"batch_{kind}_d{d}")
    E, S, rE, rS = (g[x].copy() for x in ("E0", "S0", "rE0", "rS0"))
    res = oracle.batch(kind, E, S, rE, rS, g["edges"], g["negs"], int(g["k"]), grads=True)
    assert res["loss"] == float(g["loss"])
    assert np.array_equal(res["node_ids"], g["node_ids"])
    assert np.array_equal(res["node_grads"], g["node_grads"])
    assert np.array_equal(res["rel_ids"], g["rel_ids"])
    assert np.array_equal(res["rel_grads"], g["rel_grads"])
    for got, want in ((E, "E1"), (S, "S1"), (rE, "rE1"), (rS, "rS1")):
        assert np.array_equal(got, g[want])


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n", [1, 4])
def test_epoch_matches_golden_bitwise(oracle, kind, n):
    g = golden(f"epoch_{kind}_n{n}")
    V, R, d = int(g["V"]), int(g["R"]), int(g["d"])
    E, S, rE, rS = oracle.store_init(n, V, d, R, int(g["store_seed"]))
    plan = {"states": g["states"], "bucket_order": g["bucket_order"],
            "state_offsets": g["state_offsets"]}
    res = oracle.run_epoch(g["edges"], V, R, n, plan, kind, E, S, rE, rS, dim=d,
                           batch_size=int(g["batch"]), k=int(g["k"]), seed=int(g["seed"]),
                           dumps=True)
    assert res["loss_sum"] == float(g["loss_sum"])
    assert res["edges_trained"] == int(g["edges_trained"])
    assert res["buckets_trained"] == int(g["buckets_trained"])
    for key in ("batch_loss", "batch_nodes", "batch_rels", "perm", "negs"):
        assert np.array_equal(res[key], g[key]), key
    assert np.array_equal(E, g["E"]) and np.array_equal(S, g["S"])
    if R:
        assert np.array_equal(rE, g["relE"]) and np.array_equal(rS, g["relS"])


@pytest.mark.parametrize("kind", KINDS)
def test_evaluate_matches_golden(oracle, kind):
    g = golden(f"eval_{kind}")
    mrr, hits = oracle.evaluate(kind, g["E"], g["relE"] if kind != "dot" else None, g["test"],
                                999, 10, int(g["seed"]))
    assert mrr == float(g["mrr"]) and hits == float(g["hits"])


# -------------------------------------------- reference known-answer tests
def test_loss_at_zero_scores(oracle):
    # test_train.cpp:54-81: all-zero embeddings -> every score 0, loss = P log k
    V, d, k, P = 8, 4, 2, 3
    E = np.zeros((V, d), np.float32)
    S = np.zeros((V, d), np.float32)
    edges = np.array([[0, 0xFFFFFFFF, 1], [2, 0xFFFFFFFF, 3], [4, 0xFFFFFFFF, 5]], np.uint32)
    negs = np.arange(P * k, dtype=np.uint32) % V
    res = oracle.batch("dot", E, S, None, None, edges, negs, k, grads=True)
    assert res["loss"] == pytest.approx(P * np.log(k))
    assert not res["node_grads"].any()


def test_adagrad_closed_form(oracle):
    # test_train.cpp:188-213: theta 1 -> 0.9 on g = 1, acc 0 -> 1
    V, d, k = 3, 1, 1
    E = np.array([[1.0], [0.0], [0.0]], np.float32)
    S = np.zeros((V, d), np.float32)
    # dst row 0 with src 1 = 0: gradient of dst is -IR1 = 0; use src gradient instead:
    # src 0, dst 1, neg 2 with E[1] = 1, E[2] = 0 -> g_src = w*neg - dst = -1
    E = np.array([[1.0], [1.0], [0.0]], np.float32)
    res = oracle.batch("dot", E, S, None, None, np.array([[0, 0xFFFFFFFF, 1]], np.uint32),
                       np.array([2], np.uint32), k, grads=True)
    gi = dict(zip(res["node_ids"].tolist(), res["node_grads"][:, 0].tolist()))
    assert gi[0] == -1.0
    assert E[0, 0] == pytest.approx(1.1, rel=1e-6) and S[0, 0] == 1.0


def test_finite_differences(oracle):
    # test_train.cpp:111-149: analytic gradients vs central differences
    rng = np.random.default_rng(3)
    for kind in KINDS:
        V, R, d, P, k = 20, 3, 6, 5, 3
        E = rng.uniform(-0.5, 0.5, (V, d)).astype(np.float32)
        rE = rng.uniform(-0.5, 0.5, (R, d)).astype(np.float32)
        edges = np.stack([rng.integers(0, V, P), rng.integers(0, R, P) if kind != "dot" else
                          np.full(P, 0xFFFFFFFF), rng.integers(0, V, P)], 1).astype(np.uint32)
        negs = rng.integers(0, V, P * k).astype(np.uint32)
        zS = np.zeros_like(E)
        zR = np.zeros_like(rE)
        res = oracle.batch(kind, E.copy(), zS.copy(), rE.copy(), zR.copy(), edges, negs, k,
                           apply=False, grads=True)
        node, i = int(res["node_ids"][0]), 2
        h = 1e-3
        Ep, Em = E.copy(), E.copy()
        Ep[node, i] += h
        Em[node, i] -= h
        lp = oracle.batch(kind, Ep, zS.copy(), rE.copy(), zR.copy(), edges, negs, k,
                          apply=False)["loss"]
        lm = oracle.batch(kind, Em, zS.copy(), rE.copy(), zR.copy(), edges, negs, k,
                          apply=False)["loss"]
        fd = (lp - lm) / (float(Ep[node, i]) - float(Em[node, i]))
        assert fd == pytest.approx(res["node_grads"][0, i], rel=1e-3, abs=1e-6)


def test_transe_restatement_finite_differences(oracle):
    """TransE is not in the reference (train.hpp:13): its restatement is its
    definition, so it is pinned by calculus instead -- every node and
    relation gradient against central differences of the loss."""
    rng = np.random.default_rng(4)
    V, R, d, P, k = 12, 3, 5, 6, 3
    E = rng.uniform(-0.5, 0.5, (V, d)).astype(np.float32)
    rE = rng.uniform(-0.5, 0.5, (R, d)).astype(np.float32)
    edges = np.stack([rng.integers(0, V, P), rng.integers(0, R, P), rng.integers(0, V, P)],
                     1).astype(np.uint32)
    negs = rng.integers(0, V, P * k).astype(np.uint32)
    zS, zR = np.zeros_like(E), np.zeros_like(rE)
    res = oracle.batch("transe", E.copy(), zS.copy(), rE.copy(), zR.copy(), edges, negs, k,
                       apply=False, grads=True)

    def loss(E_, rE_):
        return oracle.batch("transe", E_, zS.copy(), rE_, zR.copy(), edges, negs, k,
                            apply=False)["loss"]

    for table, ids, grads in ((0, res["node_ids"], res["node_grads"]),
                              (1, res["rel_ids"], res["rel_grads"])):
        for u, row in enumerate(ids):
            for i in range(d):
                Ep, Em, rp, rm = E.copy(), E.copy(), rE.copy(), rE.copy()
                tp, tm = (Ep, Em) if table == 0 else (rp, rm)
                tp[row, i] += 1e-3
                tm[row, i] -= 1e-3
                fd = (loss(Ep, rp) - loss(Em, rm)) / (float(tp[row, i]) - float(tm[row, i]))
                assert fd == pytest.approx(grads[u, i], rel=2e-3, abs=1e-6)


def test_transe_scores_and_zero_distance(oracle):
    # f = -||s + r - t||; an exact hit (u == t) has coefficient 0, not NaN
    E = np.array([[0.5, 0.0], [0.5, 0.0], [1.5, 0.0]], np.float32)
    rE = np.zeros((1, 2), np.float32)
    edges = np.array([[0, 0, 1]], np.uint32)
    res = oracle.batch("transe", E.copy(), np.zeros_like(E), rE.copy(), np.zeros_like(rE), edges,
                       np.array([2, 2], np.uint32), 2, apply=False, grads=True)
    # scores: pos 0, negatives -1, -1 -> loss = -(0 - (-1 + log 2))
    assert res["loss"] == pytest.approx(-(0.0 - (-1.0 + np.log(2.0))), rel=1e-15)
    assert np.isfinite(res["node_grads"]).all() and np.isfinite(res["rel_grads"]).all()


def test_random_rank_baseline(oracle):
    # test_train.cpp:312-329: random embeddings rank near H(1000)/1000 = 0.00748
    rng = np.random.default_rng(2718)
    E = rng.uniform(-0.125, 0.125, (500, 16)).astype(np.float32)
    test = np.stack([rng.integers(0, 500, 2000), np.full(2000, 0xFFFFFFFF),
                     rng.integers(0, 500, 2000)], 1).astype(np.uint32)
    mrr, _ = oracle.evaluate("dot", E, None, test, 999, 10, 1)
    base = sum(1.0 / r for r in range(1, 1001)) / 1000
    assert base / 2 < mrr < base * 2


# ------------------------------------- head-to-head with the reference lib
@pytest.mark.parametrize("kind", KINDS)
def test_random_epochs_vs_reference(oracle, reference, kind):
    rng = np.random.default_rng(11)
    for n in (1, 2, 5):
        V, R, d, Ecnt = 257, 4, 10, 3000
        edges = np.stack([rng.integers(0, V, Ecnt), rng.integers(0, R, Ecnt) if kind != "dot"
                          else np.full(Ecnt, 0xFFFFFFFF), rng.integers(0, V, Ecnt)],
                         1).astype(np.uint32)
        from oracle.oracle import single_state_plan
        plan = single_state_plan(n) if n < 4 else reference.iteration_plan(n)
        a = oracle.store_init(n, V, d, R, 9)
        b = reference.store_init(n, V, d, R, 9)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        ra = oracle.run_epoch(edges, V, R, n, plan, kind, *a, dim=d, batch_size=300, k=3,
                              seed=5, epoch=2)
        rb = reference.run_epoch(edges, V, R, n, plan, kind, *b, dim=d, batch_size=300, k=3,
                                 seed=5, epoch=2)
        assert ra["loss_sum"] == rb["loss_sum"]
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
