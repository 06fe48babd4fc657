"""Time lgd_evaluate (K6) on the TW-shaped table: 1e5 test edges x 999
candidates (developer probe; the reference evaluates 1e6 edges, PAPER.md)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2505_09258_b200 as lgd  # noqa: E402

t = bench.setup_trainer(bench.CONFIGS["tw"], 0)
rng = np.random.default_rng(5)
V = bench.CONFIGS["tw"]["nodes"]
for T in (10_000, 100_000):
    test = np.stack([rng.integers(0, V, T), rng.integers(0, 16, T), rng.integers(0, V, T)],
                    1).astype(np.uint32)
    t.evaluate(test[:1000], lgd.EvalOptions(hits_k=10, num_candidates=999, seed=1))
    t0 = time.perf_counter()
    mrr, hits = t.evaluate(test, lgd.EvalOptions(hits_k=10, num_candidates=999, seed=1))
    dt = time.perf_counter() - t0
    gb = T * 1000 * 400 / 1e9
    print(f"T={T}: {dt * 1e3:.1f} ms, {T / dt:.0f} test edges/s, {gb / dt:.0f} GB/s of candidate rows,"
          f" mrr {mrr:.5f} hits@10 {hits:.4f}")
