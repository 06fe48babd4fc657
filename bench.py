"""Benchmark of the partitioned graph-embedding training hot path on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on at
1/2/4/8 GPUs): Twitter-shaped synthetic power-law graph -- 41.6M nodes, 1.3B
edges, 16 relations -- DistMult d=100, 16 partitions, k=16 negatives per
positive, batch 100,000, lr 0.1, Adagrad eps 1e-10, seed 42.

A step is one bucket of the reference iteration plan (seeded shuffle,
negative draws and every batch of the bucket: score, sort, sparse Adagrad).
`value` is edges trained per second of device time (CUDA events), inputs
resident in HBM; `e2e` runs the same buckets through the C ABI with each
bucket's edges copied from pinned host memory and its losses read back, per
step.  `--impl reference` times the reference CPU trainer (oracle/_ref, or
the C restatement when _ref is absent) on a bounded sample of the same
workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training edges/sec per epoch (1/2/4/8 B200) and % HBM roofline vs CPU ref"
CONFIGS = {
    "tw": dict(workload="Twitter-shaped synthetic power-law graph, DistMult d=100, 16 partitions",
               nodes=41_600_000, edges=1_300_000_000, rels=16, model="distmult", dim=100, n=16),
    "lj": dict(workload="LiveJournal-shaped synthetic power-law graph, Dot d=100, 8 partitions",
               nodes=4_800_000, edges=68_000_000, rels=0, model="dot", dim=100, n=8),
    "fb15k": dict(workload="FB15k-shaped synthetic KG, DistMult d=100, 1 partition",
                  nodes=15_000, edges=592_000, rels=1345, model="distmult", dim=100, n=1),
    "fm": dict(workload="Freebase86M-shaped synthetic KG, ComplEx d=100, 32 partitions",
               nodes=86_000_000, edges=338_000_000, rels=14_800, model="complex", dim=100, n=32),
    "friendster": dict(workload="Friendster-shaped synthetic power-law graph, TransE d=128 "
                                "(one relation type: the social graph is untyped), 32 partitions",
                       nodes=65_000_000, edges=1_800_000_000, rels=1, model="transe", dim=128,
                       n=32),
}
K_NEG, BATCH, LR, SEED, ALPHA, GRAPH_SEED = 16, 100_000, 0.1, 42, 2.3, 20250509
CPU_BASELINE_BATCHES = 4  # cpu_baseline leg: 4 reference batches of P = 100,000 (~35 s)
REF_BUDGET_S = 120.0  # --impl reference: timed batches stop after ~2 min of CPU work


def peaks_tensor():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    except Exception:
        return 1590.0, "fallback"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def launch_command(argv, gpus, port):
    """`bench.py --gpus N` without a torchrun environment re-launches itself
    as N ranks (one process per GPU), exactly as the driver would."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
            os.path.abspath(__file__)] + list(argv)


def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def dist_setup(gpus, init=True):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}")
    pg = None
    if world > 1 and init:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    return rank, world, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def max_over_ranks(pg, value, local):
    if pg is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=f"cuda:{local}")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(pg, value, local):
    if pg is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=f"cuda:{local}")
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------ CPU reference
REF_BATCH = BATCH  # the reference CLI's batch (legend_main.cpp:29-38): same config as the GPU arm


def ref_workload(cfg):
    """The first bucket of the reference plan -- bucket (0,1) at position g = 0,
    pool = state 0's partitions {0,1,2} (bucket 0 / the whole graph when n = 1)
    -- of the benchmark graph, built on the host by the generator's C
    restatement (oracle/graphgen.c, bit-identical to lgd_generate_graph: see
    tests/test_gpu_graph.py), and the pool's initial rows (store init,
    store.cpp:59-86).  Loads nothing from the product package."""
    from oracle.oracle import Oracle
    lo = Oracle("restatement")
    n, V, R, d = cfg["n"], cfg["nodes"], cfg["rels"], cfg["dim"]
    stride = -(-V // n)
    bi, bj = (0, 1) if n > 1 else (0, 0)
    bucket = lo.powerlaw_bucket(V, R, cfg["edges"], ALPHA, GRAPH_SEED, n, bi, bj)
    nparts = min(3, n)
    V_loc = min(nparts * stride, V)
    E = np.zeros((V_loc, d), np.float32)
    first, count = [], []
    for p in range(nparts):
        a, b = p * stride, min((p + 1) * stride, V_loc)
        lo.init_rows(lo.derive_seed(SEED, p), b - a, d, E[a:b])
        first.append(a)
        count.append(b - a)
    S = np.zeros_like(E)
    rE = rS = None
    if R:
        rE = np.zeros((R, d), np.float32)
        lo.init_rows(lo.derive_seed(SEED, 0x52454C53), R, d, rE)
        rS = np.zeros_like(rE)
    stream = lo.derive_seed(SEED, 0x62756B74, 0, 0)  # pipeline.cpp:296, epoch 0, g = 0
    sample = (f"bucket ({bi},{bj}) of the plan (g = 0, {len(bucket):,} edges, shuffled in full), "
              f"pool {{{','.join(str(p) for p in range(nparts))}}} ({V_loc:,} rows), "
              f"{cfg['model']} d={d} k={K_NEG}, batches of {REF_BATCH:,} positives")
    return dict(bucket=bucket, first=first, count=count, E=E, S=S, rE=rE, rS=rS, stream=stream,
                sample=sample)


def cpu_sample(cfg, warmup, steps, budget_s=0.0, w=None):
    """Time the reference CPU trainer (oracle/_ref: the unmodified reference
    sources; single-threaded by design) on `warmup` + `steps` consecutive
    batches of the workload above, or fewer once `budget_s` seconds of batch
    time are spent; returns edges/s over the timed batches' wall time (each
    batch: sample_negatives + batch_loss + batch_gradients + adagrad_step)."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("reference") else "restatement"
    w = w or ref_workload(cfg)
    o = Oracle(kind)
    t0 = time.perf_counter()
    losses, extra = o.bucket_sample_batches(
        cfg["model"], w["bucket"], w["first"], w["count"], w["stream"], w["E"], w["S"], w["rE"],
        w["rS"], batch_size=REF_BATCH, k=K_NEG, max_batches=warmup + steps, budget_s=budget_s)
    wall = time.perf_counter() - t0
    nb = len(losses)
    sizes = [min(REF_BATCH, len(w["bucket"]) - b * REF_BATCH) for b in range(nb)]
    timed = range(min(warmup, nb - 1), nb)
    edges = sum(sizes[b] for b in timed)
    if kind == "reference":
        secs = sum(int(extra[b]) for b in timed) / 1e9
    else:  # the restatement reports no per-batch times: whole call, all batches
        secs, edges = wall, sum(sizes)
    return {"value": edges / secs, "unit": "edges/s", "cores": 1, "host_cores": os.cpu_count(),
            "kind": "reference" if kind == "reference" else "port",
            "sample": (w["sample"] + f": {len(timed)} timed batch(es) after "
                       f"{nb - len(timed)} warm-up, {edges:,} edges in {secs:.1f} s"),
            "seconds": secs, "edges": edges, "batches": len(timed)}


def setup_trainer(cfg, device, k=K_NEG, chunk=0):
    import paper_2505_09258_b200 as lgd
    opts = lgd.TrainOptions(learning_rate=LR, batch_size=BATCH, negatives=k, shuffle=True,
                            seed=SEED, shared_chunk=chunk)
    t = lgd.Trainer(lgd.ScoreModel(cfg["model"], cfg["dim"]), opts, device=device)
    t.generate_graph(cfg["nodes"], cfg["rels"], cfg["edges"], ALPHA, GRAPH_SEED)
    t.make_partition_plan(cfg["n"])
    t.init_store(SEED)
    return t


def reference_arm(args, cfg, rank):
    """--impl reference: the reference CPU trainer (oracle/_ref) on the same
    config -- TW-shaped DistMult d=100, n=16, P=100,000, k=16 -- one batch of
    the plan's first bucket per step, W warm-up then K timed steps.  Rank 0
    only; the product library is never loaded here."""
    if rank != 0:
        return
    # warm-up: one batch (a CPU loop has no JIT; the first batch pays the
    # table's first touch); timed: up to K batches within REF_BUDGET_S
    res = cpu_sample(cfg, min(args.warmup, 1), args.steps, budget_s=REF_BUDGET_S)
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "edges/s",
            "n_gpus": args.gpus, "steps": res["batches"], "warmup": min(args.warmup, 1),
            "ms_per_step": 1e3 * res["seconds"] / max(res["batches"], 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "num_nodes": cfg["nodes"],
                       "num_edges": cfg["edges"], "num_relations": cfg["rels"],
                       "dim": cfg["dim"], "partitions": cfg["n"], "negatives": K_NEG,
                       "batch_size": REF_BATCH, "storage": "f32 (E||S), FP64 arithmetic",
                       "graph": f"power-law alpha={ALPHA}, generator seed {GRAPH_SEED}",
                       "step": f"one batch of {REF_BATCH:,} positives of the plan's first bucket"},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "host_cores", "kind",
                                                 "sample")},
            "e2e": {"value": res["value"], "unit": "edges/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_rounds(args, cfg, rank, world, local, pg):
    """The partition-round schedule on N GPUs, through the C++
    runner (rounds.cu: lgd_train_round): a step is one round -- every rank's
    buckets of the round, then the next round's partition hand-offs as NVLink
    pulls on a side stream (overlapped with the buckets that do not touch the
    moving partitions), lock-step NCCL relation sums for typed models.  Total
    work per step is one round, so scaling is strong; N = 1 runs the same
    schedule on one rank (no hand-offs)."""
    import torch
    from paper_2505_09258_b200 import multigpu as mg
    t_setup = time.perf_counter()
    t = setup_trainer(cfg, local)
    uid = None
    if world > 1:
        box = [mg.NativeRounds.unique_id() if rank == 0 else None]
        pg.broadcast_object_list(box, src=0)
        uid = box[0]
    runner = mg.NativeRounds(t, rank, world, uid)
    R = runner.num_rounds
    setup_s = time.perf_counter() - t_setup
    unit = [0]

    def step():
        e, r = divmod(unit[0], R)
        unit[0] += 1
        return runner.run(e, r)

    for _ in range(args.warmup):
        step()
    t.reset_kernel_stats()
    t.set_profiling(True)
    clocks = Clocks(local)
    clocks.start()
    barrier(pg)
    torch.cuda.synchronize()
    edges = algo = 0.0
    dev_ms = handoff_ms = 0.0
    handoff_bytes = 0
    for _ in range(args.steps):
        res, ms, nbytes = step()
        edges += res.edges_trained
        algo += res.algorithmic_bytes
        dev_ms += res.device_ms
        handoff_ms += ms
        handoff_bytes += nbytes
    torch.cuda.synchronize()
    barrier(pg)
    clk = clocks.stop()
    launches = t.launch_count()
    stats = t.kernel_stats()
    t.set_profiling(False)
    dev_s = max_over_ranks(pg, dev_ms / 1e3, local)
    edges_all = sum_over_ranks(pg, edges, local)
    algo_all = sum_over_ranks(pg, algo, local)
    handoff_all = max_over_ranks(pg, handoff_ms, local)

    e2e = None
    if not args.no_e2e:  # the next K rounds with every bucket streamed from pinned host memory
        import paper_2505_09258_b200 as lgd
        host = lgd.PinnedArray((t.num_edges, 3), np.uint32)
        t.bucketed_edges(host.array)
        t.set_host_edges(host.array)
        step()  # one warm-up round through the host path
        barrier(pg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_edges = h2d = d2h = 0
        for _ in range(args.steps):
            res, _, _ = step()
            e_edges += res.edges_trained
            h2d += res.h2d_bytes
            d2h += res.d2h_bytes
        torch.cuda.synchronize()
        barrier(pg)
        wall = max_over_ranks(pg, time.perf_counter() - t0, local)
        t.set_host_edges(None)
        host.free()
        e2e = {"value": sum_over_ranks(pg, e_edges, local) / wall, "unit": "edges/s",
               "h2d_bytes_per_step": int(sum_over_ranks(pg, h2d, local)) // args.steps,
               "d2h_bytes_per_step": int(sum_over_ranks(pg, d2h, local)) // args.steps}
    hbm, peak_kind = peaks()
    dom = "update"
    dstat = stats[dom]
    achieved = (dstat["algorithmic_bytes"] / (dstat["total_ms"] / 1e3) / 1e9
                if dstat["total_ms"] else 0.0)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_sample(cfg, 0, CPU_BASELINE_BATCHES)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "host_cores", "kind", "sample")}
    if rank == 0:
        line = {
            "metric": METRIC, "value": edges_all / dev_s, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "num_nodes": cfg["nodes"],
                       "num_edges": cfg["edges"], "num_relations": cfg["rels"], "dim": cfg["dim"],
                       "partitions": cfg["n"], "negatives": K_NEG, "batch_size": BATCH,
                       "storage": "f32 (E||S), FP64 arithmetic",
                       "graph": f"power-law alpha={ALPHA}, generator seed {GRAPH_SEED}",
                       "schedule": "partition rounds (DESIGN.md 6): pairs of partitions per "
                                   "GPU, negative pool = the pair",
                       "step": f"one round of the partition-round schedule ({R} rounds per "
                               "epoch), all ranks", "edges_per_step": edges_all / args.steps,
                       "parallelism": (f"partition rounds over {world} GPUs, NVLink pulls on a "
                                       "side stream" + (", NCCL relation all-reduce per "
                                                        "lock-step batch" if cfg["rels"] else "")
                                       if world > 1 else "single GPU"),
                       "l2": "inputs larger than L2", "setup_s": round(setup_s, 1)},
            "roofline": {"bound": "hbm", "kernel": "segment_heads + long segments (K4), rank 0",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "peak_source": peak_kind,
                         "traffic": (traffic_from_profiles(args.config) or {}).get(dom),
                         "algorithmic_bytes_per_launch": (dstat["algorithmic_bytes"] /
                                                          max(dstat["launches"], 1)),
                         "avg_launch_ms": dstat["total_ms"] / max(dstat["launches"], 1),
                         "step_achieved": algo_all / dev_s / 1e9 / world,
                         "step_frac": algo_all / dev_s / 1e9 / world / hbm,
                         "phase_ms": {k: round(v["total_ms"], 3) for k, v in stats.items()}},
            "handoff": {"ms_per_step": handoff_all / args.steps,
                        "bytes_per_step": handoff_bytes / args.steps,
                        "note": "span of the side-stream pulls, max over ranks; overlaps compute"},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    t.close()
    if pg is not None:
        pg.destroy_process_group()


def bench_eval(args, cfg, local):
    """--eval T: K6 evaluate (train.cpp:375-412) at the workload's scale -- T
    test edges (seeded uniform, synthetic), 999 sampled candidates each,
    pessimistic ties -- timed on the device; roofline of the candidate-row
    gathers ((999 + 2 + t) rows of 4d bytes per test edge)."""
    import paper_2505_09258_b200 as lgd
    t = setup_trainer(cfg, local)
    rng = np.random.default_rng(7)
    T = args.eval
    test = np.stack([rng.integers(0, cfg["nodes"], T),
                     rng.integers(0, cfg["rels"], T) if cfg["rels"] else np.full(T, 0xFFFFFFFF),
                     rng.integers(0, cfg["nodes"], T)], 1).astype(np.uint32)
    opts = lgd.EvalOptions(hits_k=10, num_candidates=999, seed=SEED)
    t.evaluate(test[:min(T, 20000)], opts)  # warm-up
    t.reset_kernel_stats()
    t.set_profiling(True)
    wall0 = time.perf_counter()
    mrr, hits = t.evaluate(test, opts)
    wall = time.perf_counter() - wall0
    st = t.kernel_stats()["evaluate"]
    t.set_profiling(False)
    hbm, peak_kind = peaks()
    dev_s = st["total_ms"] / 1e3
    line = {"metric": "evaluate test edges/s (999 candidates, MRR / Hits@10)", "value": T / dev_s,
            "unit": "test edges/s", "n_gpus": 1, "higher_is_better": True, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["workload"], "test_edges": T,
                                             "candidates": 999, "hits_k": 10},
            "mrr": mrr, "hits_at_10": hits, "device_s": dev_s, "wall_s": wall,
            "roofline": {"bound": "hbm", "kernel": "eval_candidates + eval_score (K6)",
                         "achieved": st["algorithmic_bytes"] / dev_s / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": st["algorithmic_bytes"] / dev_s / 1e9 / hbm,
                         "peak_source": peak_kind,
                         "algorithmic_bytes": st["algorithmic_bytes"]}}
    print(json.dumps(line), flush=True)
    t.close()


def traffic_from_profiles(config):
    """ncu DRAM bytes per launch of this config's kernels (profiles/ncu_traffic.json,
    one capture per config), or None when this config was not captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(config)
    except Exception:
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="tw", choices=sorted(CONFIGS))
    ap.add_argument("--schedule", default="auto", choices=["auto", "plan", "rounds"],
                    help="rounds (default, every N): the partition-round schedule, so the "
                         "1/2/4/8-GPU points compare the same epoch; plan: the reference "
                         "iteration plan (run_epoch's 3-partition buffer; 1 GPU)")
    ap.add_argument("--eval", type=int, default=0,
                    help="T > 0: time K6 evaluate over T test edges instead of training")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--negatives", type=int, default=K_NEG,
                    help="negatives per positive (or per shared chunk)")
    ap.add_argument("--shared-chunk", type=int, default=0,
                    help="C > 0: shared-negative chunks of C positives scored on the tensor "
                         "cores (not a reference mode: no CPU baseline)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(subprocess.call(launch_command(sys.argv[1:], args.gpus, free_port())))
    if args.impl == "reference":  # CPU only: no process group
        rank, _, _, _ = dist_setup(args.gpus, init=False)
        reference_arm(args, cfg, rank)
        return
    rank, world, local, pg = dist_setup(args.gpus)
    if args.eval:
        bench_eval(args, cfg, local)
        return
    if args.warmup < 3:
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)

    schedule = args.schedule if args.schedule != "auto" else (
        "plan" if args.shared_chunk else "rounds")
    if schedule == "rounds":
        bench_rounds(args, cfg, rank, world, local, pg)
        return
    import paper_2505_09258_b200 as lgd
    t_setup = time.perf_counter()
    t = setup_trainer(cfg, local, args.negatives, args.shared_chunk)
    G = cfg["n"] ** 2
    # a step is one bucket of the plan; unit i is bucket i % G of epoch i // G
    # (small plans wrap into the next epochs).  Weak scaling: rank r trains its
    # own K consecutive units (tables replicated per GPU).
    u0 = args.warmup + rank * args.steps
    units = [(i // G, i % G) for i in range(u0, u0 + args.steps)]
    setup_s = time.perf_counter() - t_setup

    for i in range(u0 - args.warmup, u0):  # warm-up buckets (untimed)
        t.train_buckets(i // G, i % G, i % G + 1)
    t.reset_kernel_stats()
    t.set_profiling(True)
    clocks = Clocks(local)
    clocks.start()
    barrier(pg)
    t.synchronize()
    parts = [t.train_buckets(e, g, g + 1) for e, g in units]
    t.synchronize()
    barrier(pg)
    clk = clocks.stop()
    launches = t.launch_count()
    stats = t.kernel_stats()
    t.set_profiling(False)

    class _Sum:  # the timed units as one EpochResult-like record
        pass
    res = _Sum()
    for f in ("device_ms", "edges_trained", "algorithmic_bytes", "batches", "unique_nodes"):
        setattr(res, f, sum(getattr(r, f) for r in parts))

    dev_s = max_over_ranks(pg, res.device_ms / 1e3, local)
    edges_all = sum_over_ranks(pg, res.edges_trained, local)
    value = edges_all / dev_s

    # roofline of the dominant HBM-bound kernel class (per launch averages)
    hbm, peak_kind = peaks()
    cand = {k: v for k, v in stats.items() if k in ("score", "update") and v["launches"]}
    dom = max(cand, key=lambda k: cand[k]["total_ms"])
    dstat = stats[dom]
    achieved = dstat["algorithmic_bytes"] / (dstat["total_ms"] / 1e3) / 1e9
    traffic = traffic_from_profiles(args.config)
    roofline = {"bound": "hbm", "kernel": {"score": "score_kernel (K3)",
                                           "update": "segment_pass1+2 (K4)"}[dom],
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_source": peak_kind,
                "traffic": (traffic or {}).get(dom),
                "algorithmic_bytes_per_launch": dstat["algorithmic_bytes"] / dstat["launches"],
                "avg_launch_ms": dstat["total_ms"] / dstat["launches"],
                "step_achieved": res.algorithmic_bytes / (res.device_ms / 1e3) / 1e9,
                "step_frac": res.algorithmic_bytes / (res.device_ms / 1e3) / 1e9 / hbm,
                "phase_ms": {k: round(v["total_ms"], 3) for k, v in stats.items()}}

    e2e = None
    if not args.no_e2e:
        host = lgd.PinnedArray((t.num_edges, 3), np.uint32)
        t.bucketed_edges(host.array)
        for i in range(u0 - args.warmup, u0):  # warm-up calls through the host path (untimed)
            t.train_buckets_from_host(1 + i // G, i % G, i % G + 1, host.array)
        barrier(pg)
        t0 = time.perf_counter()
        h2d = d2h = 0
        for e, g in units:  # per step: H2D edges, train, D2H losses (the next epoch's streams)
            r = t.train_buckets_from_host(1 + e, g, g + 1, host.array)
            h2d += r.h2d_bytes
            d2h += r.d2h_bytes
        wall = time.perf_counter() - t0
        barrier(pg)
        wall = max_over_ranks(pg, wall, local)
        host.free()
        e2e = {"value": edges_all / wall, "unit": "edges/s",
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps}

    tensor = None
    if args.shared_chunk:  # the chunk x negatives x dim contractions on tcgen05
        sc = stats["score"]
        bf16, _ = peaks_tensor()
        flops = 6.0 * res.edges_trained * args.negatives * cfg["dim"]  # 6 P k d
        tensor = {"bound": "tensor", "kernel": "score phase: prep + gather + SG2/SG3 "
                  "(tcgen05.mma kind::tf32)", "achieved": flops / (sc["total_ms"] / 1e3) / 1e12,
                  "peak": bf16 / 2, "unit": "TFLOP/s",
                  "frac": flops / (sc["total_ms"] / 1e3) / 1e12 / (bf16 / 2),
                  "peak_source": "measured bf16 dense / 2 (TF32 rate)",
                  "flops_per_step": flops / args.steps, "score_ms": round(sc["total_ms"], 3)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and not args.shared_chunk:
        cpu = cpu_sample(cfg, 0, CPU_BASELINE_BATCHES)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "host_cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_s * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["workload"], "num_nodes": cfg["nodes"],
                       "num_edges": cfg["edges"], "num_relations": cfg["rels"],
                       "dim": cfg["dim"], "partitions": cfg["n"], "negatives": args.negatives,
                       "negatives_mode": (f"shared chunks of {args.shared_chunk} positives, "
                                          f"{args.negatives} negatives each; TF32 tensor-core "
                                          "scores, FP32 accumulate, FP64 updates"
                                          if args.shared_chunk else "independent per positive"),
                       "batch_size": BATCH, "storage": "f32 (E||S), FP64 arithmetic",
                       "graph": f"power-law alpha={ALPHA}, generator seed {GRAPH_SEED}",
                       "step": "one bucket of the reference iteration plan",
                       "buckets_timed": [[e, g] for e, g in units][:4] + (
                           [["..."]] if len(units) > 4 else []),
                       "edges_per_rank": res.edges_trained, "batches": res.batches,
                       "unique_rows_per_batch": res.unique_nodes / max(res.batches, 1),
                       "l2": (f"inputs larger than L2 ({8 * cfg['nodes'] * cfg['dim'] / 1e9:.1f} GB "
                              f"table, {12 * cfg['edges'] / 1e9:.1f} GB edges)"
                              if cfg["nodes"] * cfg["dim"] * 8 > 126e6 else
                              "table fits L2 (correctness config)"),
                       "parallelism": "bucket slices per GPU" if world > 1 else "single GPU",
                       "setup_s": round(setup_s, 1)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk,
        }
        if tensor:
            line["tensor_roofline"] = tensor
        print(json.dumps(line), flush=True)
    t.close()
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
