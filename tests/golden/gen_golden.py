"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

TEST INFRASTRUCTURE.  Runs only where /root/reference exists (the build
container): `make -C oracle ref` compiles the unmodified reference sources into
oracle/_ref/liblegend_ref.so; this script drives that library through
oracle/ref_shim.cpp and stores inputs + outputs as small .npz fixtures.  The
GPU box never sees /root/reference; tests there read these files.

    python tests/golden/gen_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle, single_state_plan  # noqa: E402

KINDS = ["dot", "distmult", "complex"]


def graph(rng, V, R, E):
    return np.stack([rng.integers(0, V, E), rng.integers(0, max(R, 1), E) if R else
                     np.full(E, 0xFFFFFFFF), rng.integers(0, V, E)], 1).astype(np.uint32)


def main():
    ref = Oracle("reference")
    out = {}

    # ---- RNG: derive_seed, raw streams, next_below incl. heavy rejection
    seeds = [(42, 0x62756B74, 0, 5), (7, 1, 2, 3), (0, 0, 0, 0), (2**64 - 1, 9, 9, 9)]
    out["rng"] = dict(
        derive_in=np.array(seeds, np.uint64),
        derive_out=np.array([ref.derive_seed(*s) for s in seeds], np.uint64),
        raw_seed=np.uint64(3919101805867400701),
        raw=ref.rng_u64(3919101805867400701, 2000),
    )
    bounds = np.array([2**63 + 1] * 200 + [5, 7, 1000, 2**32 - 1, 7800000, 1, 2**64 - 1],
                      np.uint64)
    vals, used = ref.rng_below(11, bounds)
    out["rng"].update(below_seed=np.uint64(11), below_bounds=bounds, below_vals=vals,
                      below_used=np.uint64(used))
    big = np.full(5000, 2**63 + 1, np.uint64)  # ~half of all draws reject
    bv, bu = ref.rng_below(12345, big, skip=17)
    out["rng"].update(reject_seed=np.uint64(12345), reject_skip=np.uint64(17), reject_vals=bv,
                      reject_used=np.uint64(bu))

    # ---- sampler: test_train.cpp:231-267 pool shape + a 3-range pool
    out["sampler"] = dict(
        first2=np.array([0, 100], np.uint64), count2=np.array([50, 50], np.uint64),
        s2=ref.sample_negatives([0, 100], [50, 50], 4, 2500, 4242),
        first3=np.array([0, 4000, 9000], np.uint64), count3=np.array([1000, 1000, 777], np.uint64),
        s3=ref.sample_negatives([0, 4000, 9000], [1000, 1000, 777], 16, 5000, 99, skip=12345),
    )

    # ---- partition plan (graph.cpp:120-150)
    rng = np.random.default_rng(1)
    eg = graph(rng, 1000, 3, 20000)
    stride, off, order = ref.partition_plan(eg, 1000, 7)
    out["partition"] = dict(edges=eg, V=np.uint64(1000), n=np.uint32(7), stride=np.uint64(stride),
                            offsets=off, edge_order=order)

    # ---- store init (store.cpp:59-102)
    E, S, rE, rS = ref.store_init(5, 203, 12, 7, 42)
    out["store"] = dict(n=np.uint32(5), V=np.uint64(203), dim=np.uint32(12), R=np.uint64(7),
                        seed=np.uint64(42), E=E, relE=rE)

    # ---- single batches: loss, gradients, Adagrad-updated tables
    for kind in KINDS:
        for d in (6, 12):
            rng = np.random.default_rng(100 + d)
            V, R, P, k = 60, 4, 40, 4
            E0 = rng.uniform(-0.3, 0.3, (V, d)).astype(np.float32)
            S0 = rng.uniform(0, 0.1, (V, d)).astype(np.float32)
            rE0 = rng.uniform(-0.3, 0.3, (R, d)).astype(np.float32)
            rS0 = rng.uniform(0, 0.1, (R, d)).astype(np.float32)
            edges = graph(rng, V, R if kind != "dot" else 0, P)
            negs = rng.integers(0, V, P * k).astype(np.uint32)
            E1, S1, rE1, rS1 = E0.copy(), S0.copy(), rE0.copy(), rS0.copy()
            res = ref.batch(kind, E1, S1, rE1, rS1, edges, negs, k, lr=0.1, eps=1e-10,
                            apply=True, grads=True)
            out[f"batch_{kind}_d{d}"] = dict(
                E0=E0, S0=S0, rE0=rE0, rS0=rS0, edges=edges, negs=negs, k=np.uint32(k),
                loss=np.float64(res["loss"]), node_ids=res["node_ids"],
                node_grads=res["node_grads"], rel_ids=res["rel_ids"], rel_grads=res["rel_grads"],
                E1=E1, S1=S1, rE1=rE1, rS1=rS1)

    # ---- full epochs through the reference's own in-memory restatement
    # (test_pipeline.cpp:227-269); n=1 uses the single-state convention, n=4
    # the reference plan.  The n=4 run is also checked against the real
    # on-disk run_epoch below.
    for kind in KINDS:
        for n in (1, 4):
            rng = np.random.default_rng(7 + n)
            V, R, d, Ecnt = 400, 5, 12, 6000
            edges = graph(rng, V, R if kind != "dot" else 0, Ecnt)
            plan = single_state_plan(n) if n < 4 else ref.iteration_plan(n)
            E0, S0, rE0, rS0 = ref.store_init(n, V, d, R, 42)
            E1, S1, rE1, rS1 = E0.copy(), S0.copy(), rE0.copy(), rS0.copy()
            res = ref.run_epoch(edges, V, R, n, plan, kind, E1, S1, rE1, rS1, dim=d, lr=0.1,
                                batch_size=512, k=5, shuffle=True, seed=42, epoch=0, dumps=True)
            if n >= 4:
                real = ref.run_epoch_store(edges, V, R, n, kind, dim=d, lr=0.1, batch_size=512,
                                           k=5, shuffle=True, seed=42, epoch=0, store_seed=42)
                assert real["loss_sum"] == res["loss_sum"]
                assert np.array_equal(real["E"], E1) and np.array_equal(real["S"], S1)
            out[f"epoch_{kind}_n{n}"] = dict(
                edges=edges, V=np.uint64(V), R=np.uint64(R), d=np.uint32(d), n=np.uint32(n),
                batch=np.uint32(512), k=np.uint32(5), seed=np.uint64(42), store_seed=np.uint64(42),
                states=plan["states"], bucket_order=plan["bucket_order"],
                state_offsets=plan["state_offsets"], loss_sum=np.float64(res["loss_sum"]),
                edges_trained=np.uint64(res["edges_trained"]),
                buckets_trained=np.uint64(res["buckets_trained"]), batch_loss=res["batch_loss"],
                batch_nodes=res["batch_nodes"], batch_rels=res["batch_rels"], perm=res["perm"],
                negs=res["negs"], E=E1, S=S1, relE=rE1, relS=rS1)

    # ---- evaluate (train.cpp:375-412)
    for kind in KINDS:
        rng = np.random.default_rng(5)
        V, R, d = 500, 6, 12
        Et = rng.uniform(-0.5, 0.5, (V, d)).astype(np.float32)
        rEt = rng.uniform(-0.5, 0.5, (R, d)).astype(np.float32)
        test = graph(rng, V, R if kind != "dot" else 0, 300)
        mrr, hits = ref.evaluate(kind, Et, rEt if kind != "dot" else None, test, 999, 10, 77)
        out[f"eval_{kind}"] = dict(E=Et, relE=rEt, test=test, mrr=np.float64(mrr),
                                   hits=np.float64(hits), seed=np.uint64(77))

    # ---- planner: every n in 4..40 plus the byte-stable fig6 JSON
    plans = {}
    for n in range(4, 41):
        p = ref.iteration_plan(n)
        for key in ("states", "swaps", "bucket_order", "state_offsets", "prefetch_points"):
            plans[f"n{n}_{key}"] = np.asarray(p[key])
    out["plans"] = plans
    fig6 = ref.plan_json(6)
    ref_fixture = "/root/reference/proj/tests/fixtures/fig6_plan.json"
    if os.path.exists(ref_fixture):
        assert fig6 == open(ref_fixture).read(), "reference plan_json differs from its fixture"
    with open(os.path.join(HERE, "fig6_plan.json"), "w") as f:
        f.write(fig6)

    for name, arrays in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE))
    print(f"wrote {len(out)} fixtures, {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
