import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2505_09258_b200 as lgd
from oracle.oracle import Oracle, single_state_plan
from test_gpu_shared import problem, trainer, frob
o = Oracle("restatement")
for kind in ["dot", "distmult", "complex"]:
    d, k, C, P, V, R = 100, 1000, 1000, 5000, 20000, 11
    E0, S0, rE0, edges, shared = problem(kind, d, P, V, R, k, C, 5)
    Rm = R if kind != "dot" else 0
    t = trainer(kind, d, V, Rm, edges, k, C); t.load_tables(E0, S0)
    if Rm: t.set_relations(rE0, np.zeros_like(rE0))
    negs = o.expand_shared(shared, P, k, C)
    gw = o.batch(kind, E0.copy(), S0.copy(), rE0.copy() if Rm else None, np.zeros_like(rE0) if Rm else None, edges, negs, k, apply=False, grads=True)
    gg = t.batch_gradients(edges, shared)
    # split error by contribution type: rows touched only as negatives
    print(kind, "loss rel", abs(gg["loss"]-gw["loss"])/abs(gw["loss"]), "node grad frob", frob(gg["node_grads"], gw["node_grads"]),
          "rel grad frob", frob(gg["rel_grads"], gw["rel_grads"]) if Rm else 0)
for kind in ["distmult", "complex", "dot"]:
    rng = np.random.default_rng(4)
    V, R, d, Ecnt, k, C, B = 3000, 7, 100, 40000, 200, 256, 4000
    edges = np.stack([rng.integers(0, V, Ecnt), rng.integers(0, R, Ecnt), rng.integers(0, V, Ecnt)], 1).astype(np.uint32)
    Rm = R if kind != "dot" else 0
    if not Rm: edges[:, 1] = 0xFFFFFFFF
    t = trainer(kind, d, V, Rm, edges, k, C, batch=B, n=1); t.init_store(42)
    res = t.run_epoch(0)
    E, S, rE, rS = o.store_init(1, V, d, max(R,1), 42)
    want = o.run_epoch(edges, V, Rm, 1, single_state_plan(1), kind, E, S, rE if Rm else None, rS if Rm else None, dim=d, batch_size=B, k=k, seed=42, dumps=True, chunk=C)
    Eg, Sg = t.tables()
    sc = np.maximum(np.abs(E.astype(np.float64)), 0.5/np.sqrt(d))
    print(kind, "epoch loss rel", abs(res.loss_sum-want["loss_sum"])/abs(want["loss_sum"]), "E frob", frob(Eg, E), "S frob", frob(Sg, S),
          "p99", np.quantile(np.abs(Eg.astype(np.float64)-E)/sc, 0.99), "max", (np.abs(Eg.astype(np.float64)-E)/sc).max())
