"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python profiles/sanitize_workload.py exact

exact   one epoch of every model (DistMult, ComplEx, TransE, Dot) at a small
        shape: K1 shuffle, K2 sampler, bucket presort, K3 score, K4 pass 1 + 2
        (hub segments forced by a skewed graph), the relation side pass, then
        K6 evaluate.
shared  one epoch of shared-negative chunks (tcgen05 SG2 / SG3 + K4).
Each finishes in well under a second natively; the checkers slow it ~100x.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_09258_b200 as lgd  # noqa: E402


def graph(V, R, E, seed=0):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, V, E)
    dst = rng.integers(0, V, E)
    hub = rng.random(E) < 0.2  # hub segments longer than a 32-item chunk
    dst[hub] = 7
    return np.stack([src, rng.integers(0, max(R, 1), E) if R else np.full(E, 0xFFFFFFFF), dst],
                    1).astype(np.uint32)


def run(kind, d, chunk=0, k=16):
    V, R, E = 900, 0 if kind == "dot" else 5, 6000
    opts = lgd.TrainOptions(batch_size=1000, negatives=k, seed=42, shared_chunk=chunk)
    t = lgd.Trainer(lgd.ScoreModel(kind, d), opts)
    try:
        t.set_graph(graph(V, R, E), V, R)
        t.make_partition_plan(4)
        t.init_store(42)
        res = t.run_epoch(0)
        mrr, hits = t.evaluate(graph(V, R, 200, seed=1), lgd.EvalOptions(num_candidates=99))
        print(f"{kind} d={d} chunk={chunk}: loss {res.loss_sum:.4f} mrr {mrr:.4f}", flush=True)
    finally:
        t.close()


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "exact"
    if mode == "exact":
        for kind, d in (("distmult", 100), ("complex", 100), ("transe", 128), ("dot", 36)):
            run(kind, d)
    else:
        run("distmult", 100, chunk=256, k=128)
