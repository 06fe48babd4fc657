"""Shared-negative chunks on the tensor cores (shared.cu) vs the reference
batch math on the expanded negative list (oracle).  Runs on a B200 (-m gpu).

The mode is not in the reference: every `chunk` consecutive positives share
k negatives, drawn ceil(P / chunk) * k per batch from the bucket stream.  Its
oracle is the reference batch_loss / batch_gradients / adagrad_step on the
per-positive expansion (oracle.expand_shared), in FP64.  The GPU scores in
TF32 with FP32 accumulation, so the tolerances are the FP32/TF32 ones of
SURVEY.md 8(c):
  * negative ids (sampler): bit-exact;
  * per-batch loss: |rel| <= 1e-5;
  * gradients: relative Frobenius <= 1e-3 (measured ~3e-5 .. 8e-5);
  * tables after one batch: relative Frobenius <= 5e-3 per table, and the
    99th percentile of |delta| / max(|ref|, 0.5/sqrt(d)) <= 1e-2;
  * epochs: see test_shared_epoch_matches_restatement (zero-state starts
    amplify ~1e-7 gradient differences into +-lr first steps).
"""
import numpy as np
import pytest

import paper_2505_09258_b200 as lgd

pytestmark = pytest.mark.gpu


def frob(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def assert_f32_close(got, want, d, what):
    assert frob(got, want) <= 5e-3, (what, frob(got, want))
    scale = np.maximum(np.abs(want.astype(np.float64)), 0.5 / np.sqrt(d))
    p99 = np.quantile(np.abs(got.astype(np.float64) - want) / scale, 0.99)
    assert p99 <= 1e-2, (what, p99)


def trainer(kind, d, V, R, edges, k, chunk, batch=100000, seed=42, n=1):
    opts = lgd.TrainOptions(learning_rate=0.1, batch_size=batch, negatives=k, shared_chunk=chunk,
                            seed=seed)
    t = lgd.Trainer(lgd.ScoreModel(kind, d), opts)
    t.set_graph(edges, V, R)
    t.make_partition_plan(n)
    return t


def problem(kind, d, P, V, R, k, chunk, seed):
    rng = np.random.default_rng(seed)
    E0 = rng.uniform(-0.5 / np.sqrt(d), 0.5 / np.sqrt(d), (V, d)).astype(np.float32)
    S0 = rng.uniform(0, 0.01, (V, d)).astype(np.float32)
    rE0 = rng.uniform(-0.5, 0.5, (R, d)).astype(np.float32)
    rels = rng.integers(0, R, P) if kind != "dot" else np.full(P, 0xFFFFFFFF)
    src = np.where(rng.random(P) < 0.2, 7, rng.integers(0, V, P))  # a hub
    edges = np.stack([src, rels, rng.integers(0, V, P)], 1).astype(np.uint32)
    nch = -(-P // chunk)
    shared = rng.integers(0, V, nch * k).astype(np.uint32)
    return E0, S0, rE0, edges, shared


@pytest.mark.parametrize("kind", ["dot", "distmult", "complex"])
@pytest.mark.parametrize("d,k,chunk,P,V", [
    (100, 256, 128, 1000, 5000),    # whole tiles, full chunks
    (100, 1000, 1000, 2500, 20000),  # the paper's 1e3 negatives, ragged last chunk
    (64, 100, 100, 777, 3000),      # k, chunk not multiples of the tile
    (128, 16, 50, 333, 400),        # small k: one block, heavy node reuse
    (100, 200, 300, 3000, 150),     # tiny table: negatives repeat, long segments
])
def test_shared_batch_matches_expanded_reference(oracle, kind, d, k, chunk, P, V):
    R = 11
    E0, S0, rE0, edges, shared = problem(kind, d, P, V, R, k, chunk, d + k + chunk + P)
    Rm = R if kind != "dot" else 0
    t = trainer(kind, d, V, Rm, edges, k, chunk)
    t.load_tables(E0, S0)
    if Rm:
        t.set_relations(rE0, np.zeros_like(rE0))
    negs = oracle.expand_shared(shared, P, k, chunk)
    E, S, rE, rS = E0.copy(), S0.copy(), rE0.copy(), np.zeros_like(rE0)
    gw = oracle.batch(kind, E.copy(), S.copy(), rE.copy() if Rm else None,
                      rS.copy() if Rm else None, edges, negs, k, apply=False, grads=True)
    gg = t.batch_gradients(edges, shared)
    assert gg["loss"] == pytest.approx(gw["loss"], rel=1e-5)
    assert np.array_equal(gg["node_ids"], gw["node_ids"])  # the unique-row set is exact
    assert frob(gg["node_grads"], gw["node_grads"]) <= 1e-3
    if Rm:
        assert np.array_equal(gg["rel_ids"], gw["rel_ids"])
        assert frob(gg["rel_grads"], gw["rel_grads"]) <= 1e-3
    want = oracle.batch(kind, E, S, rE if Rm else None, rS if Rm else None, edges, negs, k)
    got = t.train_batch(edges, shared)
    assert got["loss"] == pytest.approx(want["loss"], rel=1e-5)
    assert got["nodes"] == want["nodes"] and got["rels"] == want["rels"]
    Eg, Sg = t.tables()
    assert_f32_close(Eg, E, d, "E")
    assert_f32_close(Sg, S, d, "S")
    if Rm:
        rEg, _ = t.get_relations()
        assert_f32_close(rEg, rE, d, "relE")


@pytest.mark.parametrize("kind", ["dot", "distmult", "complex"])
@pytest.mark.parametrize("n", [1, 4])
@pytest.mark.parametrize("warm", [False, True])
def test_shared_epoch_matches_restatement(oracle, kind, n, warm):
    """Full epochs: per-bucket shuffles and the ceil(P/C) k shared draws per
    batch come from the bucket stream bit-exactly (unique-row counts match);
    the loss within 1e-5.  Tables: from the store's zero Adagrad state the
    first step of every element is +-lr whatever |g| is (train.cpp:351-352),
    so elements whose first gradient cancels to ~1e-7 can take the opposite
    sign under any non-FP64 arithmetic (SURVEY 8(c) calibration), and a
    flipped element (a 0.2 step on a 0.05 weight) changes every later score
    it enters: the cold start is chaotic at lr 0.1 on this small, densely
    reused table.  It is held to the loss / index bounds and a loose 0.3
    Frobenius sanity bound; the warm start (state preloaded with 1e-2, so
    steps scale with |g|) is held to relative Frobenius 1e-3 and p99 1e-3."""
    rng = np.random.default_rng(3 + n)
    V, R, d, Ecnt, k, C, B = 3000, 7, 100, 40000, 200, 256, 4000
    Rm = R if kind != "dot" else 0
    rels = rng.integers(0, R, Ecnt) if Rm else np.full(Ecnt, 0xFFFFFFFF)
    edges = np.stack([rng.integers(0, V, Ecnt), rels, rng.integers(0, V, Ecnt)],
                     1).astype(np.uint32)
    t = trainer(kind, d, V, Rm, edges, k, C, batch=B, n=n)
    t.init_store(42)
    E, S, rE, rS = oracle.store_init(n, V, d, max(R, 1), 42)
    if warm:
        S[:] = 1e-2
        t.load_tables(E, S)
    res = t.run_epoch(0)
    from oracle.oracle import single_state_plan
    plan = single_state_plan(n) if n < 4 else _plan_arrays(lgd.plan_iteration_order(n))
    want = oracle.run_epoch(edges, V, Rm, n, plan, kind, E, S, rE if Rm else None,
                            rS if Rm else None, dim=d, batch_size=B, k=k, seed=42, dumps=True,
                            chunk=C)
    assert res.edges_trained == want["edges_trained"] == Ecnt
    assert res.unique_nodes == int(want["batch_nodes"].sum())
    assert res.loss_sum == pytest.approx(want["loss_sum"], rel=1e-5)
    Eg, Sg = t.tables()
    if warm:
        assert frob(Eg, E) <= 1e-3 and frob(Sg, S) <= 1e-3, (frob(Eg, E), frob(Sg, S))
        scale = np.maximum(np.abs(E.astype(np.float64)), 0.5 / np.sqrt(d))
        assert np.quantile(np.abs(Eg - E.astype(np.float64)) / scale, 0.99) <= 1e-3
    else:
        assert np.isfinite(Eg).all() and frob(Eg, E) <= 0.3 and frob(Sg, S) <= 0.3
    if Rm:
        rEg, _ = t.get_relations()
        assert frob(rEg, rE) <= (1e-3 if warm else 0.3)


def _plan_arrays(plan):
    return dict(states=plan.states, bucket_order=plan.bucket_order,
                state_offsets=plan.state_offsets)


def test_shared_mode_rejects_unsupported_shapes():
    """TransE and dimensions off the 16-byte rows / 128 TMEM columns are
    refused when the options are set (lgd_create, lgd_set_options)."""
    edges = np.array([[0, 0, 1], [1, 0, 2]], np.uint32)
    with pytest.raises(lgd.InvalidArgument, match="shared-negative"):
        trainer("transe", 16, 10, 2, edges, 4, 2)
    with pytest.raises(lgd.InvalidArgument, match="shared-negative"):
        trainer("distmult", 6, 10, 2, edges, 4, 2)  # d % 4 != 0
    with pytest.raises(lgd.InvalidArgument, match="shared-negative"):
        trainer("dot", 132, 10, 0, edges, 4, 2)  # more than 128 TMEM columns


@pytest.mark.parametrize("kind", ["dot", "distmult"])
def test_shared_online_softmax_rescales(oracle, kind):
    """SG2's online softmax moves its reference max, and rescales the mix
    accumulator, only when a later 128-negative block's max exceeds it by more
    than 2^8 in weight.  Shared negatives whose last blocks hold rows ~300x
    larger force such rescales; the same negatives with the large rows first
    need none.  The two orders give the same loss and gradients (the softmax
    is order-free; FP32 sums in another order), and both match the expanded
    reference within TF32 tolerances scaled to the large scores."""
    d, k, chunk, P, V, R = 64, 1000, 256, 1024, 4000, 5
    rng = np.random.default_rng(17)
    E0 = rng.uniform(-0.5 / np.sqrt(d), 0.5 / np.sqrt(d), (V, d)).astype(np.float32)
    E0[V // 2:] *= 300.0  # the large rows: only ever shared negatives
    S0 = rng.uniform(0, 0.01, (V, d)).astype(np.float32)
    rE0 = rng.uniform(0.5, 1.0, (R, d)).astype(np.float32)
    Rm = R if kind != "dot" else 0
    rels = rng.integers(0, R, P) if Rm else np.full(P, 0xFFFFFFFF)
    edges = np.stack([rng.integers(0, V // 2, P), rels, rng.integers(0, V // 2, P)],
                     1).astype(np.uint32)
    nch = -(-P // chunk)
    small = rng.integers(0, V // 2, (nch, 512))
    large = rng.integers(V // 2, V, (nch, k - 512))
    orders = {"large last (rescales)": np.concatenate([small, large], 1),
              "large first": np.concatenate([large, small], 1)}
    got = {}
    for name, sh in orders.items():
        shared = sh.reshape(-1).astype(np.uint32)
        t = trainer(kind, d, V, Rm, edges, k, chunk)
        t.load_tables(E0, S0)
        if Rm:
            t.set_relations(rE0, np.zeros_like(rE0))
        got[name] = t.batch_gradients(edges, shared)
        negs = oracle.expand_shared(shared, P, k, chunk)
        want = oracle.batch(kind, E0.copy(), S0.copy(), rE0.copy() if Rm else None,
                            np.zeros_like(rE0) if Rm else None, edges, negs, k, apply=False,
                            grads=True)
        g = got[name]
        assert g["loss"] == pytest.approx(want["loss"], rel=1e-3), name
        assert np.array_equal(g["node_ids"], want["node_ids"]), name
        assert frob(g["node_grads"], want["node_grads"]) <= 1e-2, name
        t.close()
    a, b = got.values()
    assert a["loss"] == pytest.approx(b["loss"], rel=1e-5)
    assert np.array_equal(a["node_ids"], b["node_ids"])
    assert frob(a["node_grads"], b["node_grads"]) <= 1e-4
