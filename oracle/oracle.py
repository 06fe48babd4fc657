"""ctypes bindings for the test-only oracles.  TEST INFRASTRUCTURE ONLY.

Two libraries share one C signature set (prefix ``lo_`` / ``ref_``):

* ``Oracle("restatement")`` -> oracle/liblegend_oracle.so, the plain-C
  restatement of the reference hot path (oracle/legend_oracle.c).  Travels to
  the GPU box; the -m gpu parity tests check the CUDA path against it.
* ``Oracle("reference")``   -> oracle/_ref/liblegend_ref.so, the unmodified
  reference sources compiled by oracle/Makefile (plus oracle/ref_shim.cpp).
  Used to generate tests/golden/ and to pin the restatement.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "restatement": os.path.join(HERE, "liblegend_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "liblegend_ref.so"),
}
ERRORS = {1: ValueError, 2: RuntimeError, 3: IndexError, 4: MemoryError}

u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
KINDS = {"dot": 0, "distmult": 1, "complex": 2, "transe": 3}


def available(which: str) -> bool:
    return os.path.exists(PATHS[which])


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Oracle:
    def __init__(self, which: str = "restatement"):
        self.which = which
        self.pre = "lo_" if which == "restatement" else "ref_"
        self.lib = C.CDLL(PATHS[which])
        L, p = self.lib, self.pre
        vp, u64, u32, i32, f64 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
        self._fn = {}

        def bind(name, res, args):
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
            self._fn[name] = f

        bind("derive_seed", u64, [u64, u64, u64, u64])
        bind("rng_u64", None, [u64, u64, u64, vp])
        bind("rng_below_seq", None, [u64, u64, vp, u64, vp, vp])
        bind("partition_plan", i32, [vp, u64, u64, u32, vp, vp, vp])
        bind("sample_negatives", i32, [vp, vp, i32, u32, u64, u64, u64, vp])
        bind("batch", i32, [i32, u32, vp, vp, u64, vp, vp, u64, vp, u64, vp, u32, f64, f64, i32,
                            vp, vp, vp, vp, vp, vp, vp])
        bind("evaluate", i32, [i32, u32, vp, u64, vp, u64, vp, u64, u32, u32, u64, vp, vp])
        bind("bucket_sample", i32, [vp, u64, vp, vp, i32, u64, i32, u32, u32, u64, i32, u32, vp,
                                    vp, u64, vp, vp, u64, f64, f64, vp, vp])
        if which == "restatement":
            bind("bucket_sample_ex", i32, [vp, u64, vp, vp, i32, u64, i32, u32, u32, u64, i32,
                                           u32, vp, vp, u64, vp, vp, u64, f64, f64, vp, vp, vp,
                                           vp])
            bind("det_pow", f64, [f64, f64])
            bind("det_log", f64, [f64])
            bind("det_exp", f64, [f64])
            bind("powerlaw_edges", i32, [u64, u64, f64, u64, u64, u64, vp])
            bind("powerlaw_bucket", i32, [u64, u64, u64, f64, u64, u32, u32, u32, i32, vp, u64,
                                          vp])
            bind("shuffle_perm", None, [u64, u64, vp, vp])
            bind("batch_split", i32, [i32, u32, vp, vp, u64, vp, vp, u64, vp, u64, vp, u32, f64,
                                      f64, i32, i32, vp, vp, vp, vp])
            bind("adagrad_touched", None, [vp, vp, vp, u64, u32, f64, f64])
            bind("run_rounds", i32, [vp, u64, u64, u64, u32, vp, u64, u32, i32, u32, f64, f64,
                                     u32, u32, i32, u64, u32, vp, vp, vp, vp, vp, vp])
            bind("store_init", None, [u32, u64, u32, u64, u64, vp, vp, vp, vp])
            bind("run_epoch_ex", i32, [vp, u64, u64, u64, u32, u64, vp, vp, u64, vp, vp, vp,
                                       i32, u32, f64, f64, u32, u32, u32, i32, u64, u32, vp, vp,
                                       vp, vp, vp, vp, vp, vp, u64, vp, vp, vp, vp, vp])
            bind("expand_shared", i32, [vp, u64, u32, u32, vp])
        else:
            bind("store_init", i32, [C.c_char_p, u32, u64, u32, u64, u64, vp, vp, vp, vp])
            bind("run_epoch_inmem", i32, [vp, u64, u64, u64, u32, u64, vp, vp, vp, i32, u32, f64,
                                          f64, u32, u32, i32, u64, u32, vp, vp, vp, vp, vp, vp,
                                          vp, vp, u64, vp, vp, vp, vp, vp])
            bind("run_epoch_store", i32, [C.c_char_p, vp, u64, u64, u64, u32, i32, u32, f64, f64,
                                          u32, u32, i32, u64, u32, u64, vp, vp, vp, vp, vp, vp,
                                          vp])
            bind("iteration_plan", i32, [u32, u64, vp, vp, vp, vp, vp, vp])
            bind("plan_json", i32, [u32, C.c_char_p, u64, vp])
            bind("verify_prefetchable", i32, [u32, u64, vp, vp, vp, vp, vp, vp])
            bind("last_error", C.c_char_p, [])
            bind("bucket_sample_timed", i32, [vp, u64, vp, vp, i32, u64, i32, u32, u32, u64,
                                              i32, u32, vp, vp, u64, vp, vp, u64, f64, f64, vp,
                                              vp, vp, u64])
            bind("write_graph", i32, [C.c_char_p, vp, u64, u64, u64])
            bind("ingest", i32, [C.c_char_p, i32, i32, vp, u64, vp, vp, vp])
            bind("read_graph", i32, [C.c_char_p, vp, u64, vp, vp, vp])

    def _check(self, rc):
        if rc:
            msg = ""
            if "last_error" in self._fn:
                msg = self._fn["last_error"]().decode()
            raise ERRORS.get(rc, RuntimeError)(f"{self.which} oracle error {rc}: {msg}")

    # ------------------------------------------------- synthetic graphs
    def powerlaw_edges(self, num_nodes, num_rels, alpha, seed, begin, end):
        """Edges [begin, end) of the benchmark's power-law graph (graphgen.c),
        bit-identical to lgd_generate_graph's (restatement only)."""
        out = np.zeros((max(end - begin, 1), 3), np.uint32)
        self._check(self._fn["powerlaw_edges"](num_nodes, num_rels, alpha, seed, begin, end,
                                               _ptr(out)))
        return out[:end - begin]

    def powerlaw_bucket(self, num_nodes, num_rels, num_edges, alpha, seed, n, bi, bj,
                        threads=None):
        """Bucket (bi, bj) of make_partition_plan(graph, n) of the power-law
        graph, in ingest order, scanned with `threads` host threads."""
        threads = threads or os.cpu_count() or 1
        cnt = np.zeros(1, np.uint64)
        self._check(self._fn["powerlaw_bucket"](num_nodes, num_rels, num_edges, alpha, seed, n,
                                                bi, bj, threads, None, 0, _ptr(cnt)))
        out = np.zeros((max(int(cnt[0]), 1), 3), np.uint32)
        self._check(self._fn["powerlaw_bucket"](num_nodes, num_rels, num_edges, alpha, seed, n,
                                                bi, bj, threads, _ptr(out), int(cnt[0]),
                                                _ptr(cnt)))
        return out[:int(cnt[0])]

    # ---------------------------------------------------------------- RNG
    def derive_seed(self, base, a, b=0, c=0):
        return int(self._fn["derive_seed"](base, a, b, c))

    def rng_u64(self, seed, n, skip=0):
        out = np.zeros(n, np.uint64)
        self._fn["rng_u64"](seed, skip, n, _ptr(out))
        return out

    def rng_below(self, seed, bounds, skip=0):
        bounds = np.ascontiguousarray(bounds, np.uint64)
        out = np.zeros(len(bounds), np.uint64)
        used = np.zeros(1, np.uint64)
        self._fn["rng_below_seq"](seed, skip, _ptr(bounds), len(bounds), _ptr(out), _ptr(used))
        return out, int(used[0])

    # --------------------------------------------------------- partitions
    def partition_plan(self, edges, num_nodes, n):
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        E = len(edges)
        stride = np.zeros(1, np.uint64)
        offsets = np.zeros(n * n + 1, np.uint64)
        order = np.zeros(max(E, 1), np.uint64)
        self._check(self._fn["partition_plan"](_ptr(edges), E, num_nodes, n, _ptr(stride),
                                               _ptr(offsets), _ptr(order)))
        return int(stride[0]), offsets, order[:E]

    def store_init(self, n, num_nodes, dim, num_rels, seed):
        E = np.zeros((num_nodes, dim), np.float32)
        S = np.zeros((num_nodes, dim), np.float32)
        rE = np.zeros((max(num_rels, 1), dim), np.float32)
        rS = np.zeros((max(num_rels, 1), dim), np.float32)
        if self.which == "restatement":
            self._fn["store_init"](n, num_nodes, dim, num_rels, seed, _ptr(E), _ptr(S), _ptr(rE),
                                   _ptr(rS))
        else:
            with tempfile.TemporaryDirectory() as d:
                self._check(self._fn["store_init"](os.path.join(d, "s").encode(), n, num_nodes,
                                                   dim, num_rels, seed, _ptr(E), _ptr(S),
                                                   _ptr(rE), _ptr(rS)))
        return E, S, rE[:num_rels], rS[:num_rels]

    def sample_negatives(self, first, count, k, num_positives, seed, skip=0):
        first = np.ascontiguousarray(first, np.uint64)
        count = np.ascontiguousarray(count, np.uint64)
        out = np.zeros(max(num_positives * k, 1), np.uint32)
        self._check(self._fn["sample_negatives"](_ptr(first), _ptr(count), len(first), k,
                                                 num_positives, seed, skip, _ptr(out)))
        return out[:num_positives * k]

    def shuffle_perm(self, seed, m):
        """pipeline.cpp:297-301 on positions (restatement only)."""
        perm = np.zeros(max(m, 1), np.uint32)
        used = np.zeros(1, np.uint64)
        self._fn["shuffle_perm"](seed, m, _ptr(perm), _ptr(used))
        return perm[:m], int(used[0])

    # ---------------------------------------------------------- training
    def batch(self, kind, E, S, relE, relS, edges, negs, k, lr=0.1, eps=1e-10, apply=True,
              grads=False):
        """One batch_loss + batch_gradients (+ adagrad_step if apply), in place."""
        kind = KINDS.get(kind, kind)
        V, d = E.shape
        R = relE.shape[0] if relE is not None else 0
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        negs = np.ascontiguousarray(negs, np.uint32)
        P = len(edges)
        loss = np.zeros(1, np.float64)
        nn = np.zeros(1, np.uint64)
        nr = np.zeros(1, np.uint64)
        cap = P * (k + 2) + 1
        ids = np.zeros(cap, np.uint32) if grads else None
        g = np.zeros((cap, d), np.float64) if grads else None
        rids = np.zeros(P + 1, np.uint32) if grads else None
        rg = np.zeros((P + 1, d), np.float64) if grads else None
        if relE is None:
            relE = np.zeros((0, d), np.float32)
            relS = np.zeros((0, d), np.float32)
        self._check(self._fn["batch"](kind, d, _ptr(E), _ptr(S), V, _ptr(relE), _ptr(relS), R,
                                      _ptr(edges), P, _ptr(negs), k, lr, eps, int(apply),
                                      _ptr(loss), _ptr(nn), _ptr(ids), _ptr(g), _ptr(nr),
                                      _ptr(rids), _ptr(rg)))
        out = {"loss": float(loss[0]), "nodes": int(nn[0]), "rels": int(nr[0])}
        if grads:
            out.update(node_ids=ids[:out["nodes"]].copy(), node_grads=g[:out["nodes"]].copy(),
                       rel_ids=rids[:out["rels"]].copy(), rel_grads=rg[:out["rels"]].copy())
        return out

    def run_epoch(self, edges, num_nodes, num_rels, n, plan, kind, E, S, relE, relS, *, dim,
                  lr=0.1, eps=1e-10, batch_size=100000, k=16, shuffle=True, seed=42, epoch=0,
                  dumps=False, chunk=0):
        """All-resident real-train epoch under `plan` (see plan_arrays), in place.
        chunk > 0: shared-negative chunks (restatement only; k negatives per
        chunk of `chunk` positives, expanded onto the reference batch math)."""
        kind = KINDS.get(kind, kind)
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        Ecount = len(edges)
        states = np.ascontiguousarray(plan["states"], np.uint32)
        order = np.ascontiguousarray(plan["bucket_order"], np.uint32)
        soff = np.ascontiguousarray(plan["state_offsets"], np.uint64)
        S_ = len(states)
        maxb = Ecount // max(batch_size, 1) + n * n + 1
        loss = np.zeros(1, np.float64)
        et = np.zeros(1, np.uint64)
        bt = np.zeros(1, np.uint64)
        nb = np.zeros(1, np.uint64)
        bl = np.zeros(maxb, np.float64) if dumps else None
        bn = np.zeros(maxb, np.uint64) if dumps else None
        br = np.zeros(maxb, np.uint64) if dumps else None
        pd = np.zeros(max(Ecount, 1), np.uint32) if dumps else None
        nd = np.zeros(max(Ecount * k, 1), np.uint32) if dumps else None
        if relE is None or len(relE) == 0:
            relE = np.zeros((1, dim), np.float32)
            relS = np.zeros((1, dim), np.float32)
        if self.which == "restatement":
            stride, offsets, eorder = self.partition_plan(edges, num_nodes, n)
            rc = self._fn["run_epoch_ex"](
                _ptr(edges), Ecount, num_nodes, num_rels, n, stride, _ptr(offsets), _ptr(eorder),
                S_, _ptr(states), _ptr(order), _ptr(soff), kind, dim, lr, eps, batch_size, k,
                chunk, int(shuffle), seed, epoch, _ptr(E), _ptr(S), _ptr(relE), _ptr(relS), _ptr(loss),
                _ptr(et), _ptr(bt), _ptr(nb), maxb, _ptr(bl), _ptr(bn), _ptr(br), _ptr(pd),
                _ptr(nd))
        else:
            assert chunk == 0, "shared-negative chunks are not a reference mode"
            rc = self._fn["run_epoch_inmem"](
                _ptr(edges), Ecount, num_nodes, num_rels, n, S_, _ptr(states), _ptr(order),
                _ptr(soff), kind, dim, lr, eps, batch_size, k, int(shuffle), seed, epoch, _ptr(E),
                _ptr(S), _ptr(relE), _ptr(relS), _ptr(loss), _ptr(et), _ptr(bt), _ptr(nb), maxb,
                _ptr(bl), _ptr(bn), _ptr(br), _ptr(pd), _ptr(nd))
        self._check(rc)
        out = {"loss_sum": float(loss[0]), "edges_trained": int(et[0]),
               "buckets_trained": int(bt[0]), "num_batches": int(nb[0])}
        if dumps:
            b = out["num_batches"]
            out.update(batch_loss=bl[:b].copy(), batch_nodes=bn[:b].copy(),
                       batch_rels=br[:b].copy(), perm=pd[:Ecount].copy(),
                       negs=nd[:out["edges_trained"] * k].copy() if not chunk else nd)
        return out

    def expand_shared(self, shared, cnt, k, chunk):
        """[ceil(cnt/chunk) * k] shared draws -> the [cnt * k] per-positive list."""
        shared = np.ascontiguousarray(shared, np.uint32)
        out = np.zeros(cnt * k, np.uint32)
        self._check(self._fn["expand_shared"](_ptr(shared), cnt, k, chunk, _ptr(out)))
        return out

    def bucket_sample(self, kind, bucket_edges, first, count, stream_seed, E, S, relE, relS, *,
                      batch_size, k, max_batches, shuffle=True, lr=0.1, eps=1e-10):
        """One bucket of the real-train loop, at most max_batches batches, in place."""
        kind = KINDS.get(kind, kind)
        V, d = E.shape
        R = relE.shape[0] if relE is not None else 0
        if relE is None:
            relE = np.zeros((1, d), np.float32)
            relS = np.zeros((1, d), np.float32)
        be = np.ascontiguousarray(bucket_edges, np.uint32).reshape(-1, 3)
        first = np.ascontiguousarray(first, np.uint64)
        count = np.ascontiguousarray(count, np.uint64)
        loss = np.zeros(1, np.float64)
        done = np.zeros(1, np.uint64)
        self._check(self._fn["bucket_sample"](
            _ptr(be), len(be), _ptr(first), _ptr(count), len(first), stream_seed, int(shuffle),
            batch_size, k, max_batches, kind, d, _ptr(E), _ptr(S), V, _ptr(relE), _ptr(relS), R,
            lr, eps, _ptr(loss), _ptr(done)))
        return float(loss[0]), int(done[0])

    def bucket_sample_batches(self, kind, bucket_edges, first, count, stream_seed, E, S, relE,
                              relS, *, batch_size, k, max_batches, shuffle=True, lr=0.1,
                              eps=1e-10, budget_s=0.0):
        """bucket_sample with per-batch outputs.  Restatement: (losses, unique
        nodes per batch); reference: (losses, wall ns per batch), stopping once
        budget_s > 0 seconds of batch time are spent.  In place."""
        kind = KINDS.get(kind, kind)
        V, d = E.shape
        R = relE.shape[0] if relE is not None else 0
        if relE is None:
            relE = np.zeros((1, d), np.float32)
            relS = np.zeros((1, d), np.float32)
        be = np.ascontiguousarray(bucket_edges, np.uint32).reshape(-1, 3)
        first = np.ascontiguousarray(first, np.uint64)
        count = np.ascontiguousarray(count, np.uint64)
        losses = np.zeros(max(max_batches, 1), np.float64)
        extra = np.zeros(max(max_batches, 1), np.uint64)
        done = np.zeros(1, np.uint64)
        if self.which == "restatement":
            total = np.zeros(1, np.float64)
            self._check(self._fn["bucket_sample_ex"](
                _ptr(be), len(be), _ptr(first), _ptr(count), len(first), stream_seed,
                int(shuffle), batch_size, k, max_batches, kind, d, _ptr(E), _ptr(S), V,
                _ptr(relE), _ptr(relS), R, lr, eps, _ptr(total), _ptr(done), _ptr(losses),
                _ptr(extra)))
            nb = -(-int(done[0]) // batch_size) if done[0] else 0
        else:
            self._check(self._fn["bucket_sample_timed"](
                _ptr(be), len(be), _ptr(first), _ptr(count), len(first), stream_seed,
                int(shuffle), batch_size, k, max_batches, kind, d, _ptr(E), _ptr(S), V,
                _ptr(relE), _ptr(relS), R, lr, eps, _ptr(losses), _ptr(extra), _ptr(done),
                int(budget_s * 1e9)))
            nb = int(done[0])
        return losses[:nb], extra[:nb]

    def write_graph(self, directory, edges, num_nodes, num_relations=0):
        """write_graph (graph.cpp:152-171) of the reference itself."""
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        self._check(self._fn["write_graph"](os.fsencode(directory), _ptr(edges), len(edges),
                                            num_nodes, num_relations))

    def ingest(self, path, triples=True, remap_ids=False):
        """ingest (graph.cpp:39-118) of the reference itself."""
        cnt, V, R = (np.zeros(1, np.uint64) for _ in range(3))
        p = os.fsencode(path)
        self._check(self._fn["ingest"](p, int(triples), int(remap_ids), None, 0, _ptr(cnt),
                                       _ptr(V), _ptr(R)))
        out = np.zeros((max(int(cnt[0]), 1), 3), np.uint32)
        self._check(self._fn["ingest"](p, int(triples), int(remap_ids), _ptr(out), int(cnt[0]),
                                       _ptr(cnt), _ptr(V), _ptr(R)))
        return out[:int(cnt[0])], int(V[0]), int(R[0])

    def read_graph(self, directory):
        """read_graph (graph.cpp:173-192) of the reference itself."""
        cnt, V, R = (np.zeros(1, np.uint64) for _ in range(3))
        d = os.fsencode(directory)
        self._check(self._fn["read_graph"](d, None, 0, _ptr(cnt), _ptr(V), _ptr(R)))
        out = np.zeros((max(int(cnt[0]), 1), 3), np.uint32)
        self._check(self._fn["read_graph"](d, _ptr(out), int(cnt[0]), _ptr(cnt), _ptr(V),
                                           _ptr(R)))
        return out[:int(cnt[0])], int(V[0]), int(R[0])

    def init_rows(self, stream_seed, rows, dim, out):
        """fill_uniform_rows (store.cpp:19-25) into a float32 slice (restatement)."""
        self.lib.lo_init_rows.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_void_p]
        self.lib.lo_init_rows(stream_seed, rows, dim, _ptr(out))

    def batch_nodes_only(self, kind, E, S, relE, relS, edges, negs, k, lr=0.1, eps=1e-10):
        """batch_loss + batch_gradients; node Adagrad applied, relation
        gradients returned as a dense [R x (d+1)] array (last column: touched)."""
        kind = KINDS.get(kind, kind)
        V, d = E.shape
        R = relE.shape[0] if relE is not None else 0
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        negs = np.ascontiguousarray(negs, np.uint32)
        P = len(edges)
        loss = np.zeros(1, np.float64)
        nr = np.zeros(1, np.uint64)
        rids = np.zeros(P + 1, np.uint32)
        rg = np.zeros((P + 1, d), np.float64)
        if relE is None:
            relE = np.zeros((1, d), np.float32)
            relS = np.zeros((1, d), np.float32)
        self._check(self._fn["batch_split"](kind, d, _ptr(E), _ptr(S), V, _ptr(relE), _ptr(relS),
                                            R, _ptr(edges), P, _ptr(negs), k, lr, eps, 1, 0,
                                            _ptr(loss), _ptr(nr), _ptr(rids), _ptr(rg)))
        dense = np.zeros((max(R, 1), d + 1), np.float64)
        n = int(nr[0])
        dense[rids[:n], :d] = rg[:n]
        dense[rids[:n], d] = 1.0
        return float(loss[0]), dense

    def adagrad_touched(self, relE, relS, summed, lr=0.1, eps=1e-10):
        R, d = relE.shape
        summed = np.ascontiguousarray(summed, np.float64)
        self._fn["adagrad_touched"](_ptr(relE), _ptr(relS), _ptr(summed), R, d, lr, eps)

    def run_rounds(self, edges, num_nodes, num_rels, n, items, num_ranks, kind, E, S, relE, relS,
                   *, dim, lr=0.1, eps=1e-10, batch_size=100000, k=16, shuffle=True, seed=42,
                   epoch=0):
        """Serialized multi-GPU round schedule (lock-step relation sums), in place.
        items: (count, 8) u64 rows (src, dst, g, pool0, pool1, pool2, round, pair)."""
        kind = KINDS.get(kind, kind)
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        items = np.ascontiguousarray(items, np.uint64).reshape(-1, 8)
        if relE is None or len(relE) == 0:
            relE = np.zeros((1, dim), np.float32)
            relS = np.zeros((1, dim), np.float32)
        loss = np.zeros(1, np.float64)
        et = np.zeros(1, np.uint64)
        self._check(self._fn["run_rounds"](_ptr(edges), len(edges), num_nodes, num_rels, n,
                                           _ptr(items), len(items), num_ranks, kind, dim, lr, eps,
                                           batch_size, k, int(shuffle), seed, epoch, _ptr(E),
                                           _ptr(S), _ptr(relE), _ptr(relS), _ptr(loss), _ptr(et)))
        return {"loss_sum": float(loss[0]), "edges_trained": int(et[0])}

    def evaluate(self, kind, E, relE, test_edges, num_candidates=999, hits_k=10, seed=0):
        kind = KINDS.get(kind, kind)
        V, d = E.shape
        relE = relE if relE is not None and len(relE) else np.zeros((0, d), np.float32)
        test_edges = np.ascontiguousarray(test_edges, np.uint32).reshape(-1, 3)
        mrr = np.zeros(1, np.float64)
        hits = np.zeros(1, np.float64)
        self._check(self._fn["evaluate"](kind, d, _ptr(E), V, _ptr(relE), len(relE),
                                         _ptr(test_edges), len(test_edges), num_candidates,
                                         hits_k, seed, _ptr(mrr), _ptr(hits)))
        return float(mrr[0]), float(hits[0])

    # ---------------------------------------------- reference-only helpers
    def iteration_plan(self, n):
        assert self.which == "reference"
        S = np.zeros(1, np.uint64)
        z = np.zeros(1, np.uint64)
        self._check(self._fn["iteration_plan"](n, 0, _ptr(S), None, None, None, None, None))
        s = int(S[0])
        states = np.zeros((s, 3), np.uint32)
        swaps = np.zeros((max(s - 1, 1), 2), np.uint32)
        order = np.zeros((n * n, 2), np.uint32)
        soff = np.zeros(s + 1, np.uint64)
        pre = np.zeros(max(s - 1, 1), np.uint64)
        self._check(self._fn["iteration_plan"](n, s, _ptr(z), _ptr(states), _ptr(swaps),
                                               _ptr(order), _ptr(soff), _ptr(pre)))
        return {"n": n, "states": states, "swaps": swaps[:s - 1], "bucket_order": order,
                "state_offsets": soff, "prefetch_points": pre[:s - 1]}

    def plan_json(self, n):
        ln = np.zeros(1, np.uint64)
        self._check(self._fn["plan_json"](n, None, 0, _ptr(ln)))
        buf = C.create_string_buffer(int(ln[0]) + 1)
        self._check(self._fn["plan_json"](n, buf, int(ln[0]) + 1, _ptr(ln)))
        return buf.value.decode()

    def verify_prefetchable(self, plan):
        n = plan["n"]
        st = np.ascontiguousarray(plan["states"], np.uint32)
        sw = np.ascontiguousarray(plan["swaps"], np.uint32)
        bo = np.ascontiguousarray(plan["bucket_order"], np.uint32)
        so = np.ascontiguousarray(plan["state_offsets"], np.uint64)
        pp = np.ascontiguousarray(plan["prefetch_points"], np.uint64)
        ok = np.zeros(1, np.int32)
        self._check(self._fn["verify_prefetchable"](n, len(st), _ptr(st), _ptr(sw), _ptr(bo),
                                                    _ptr(so), _ptr(pp), _ptr(ok)))
        return bool(ok[0])

    def run_epoch_store(self, edges, num_nodes, num_rels, n, kind, *, dim, lr=0.1, eps=1e-10,
                        batch_size=100000, k=16, shuffle=True, seed=42, epoch=0, store_seed=42):
        """The real run_epoch (pipeline.cpp:215) over an on-disk store (n >= 4)."""
        assert self.which == "reference"
        kind = KINDS.get(kind, kind)
        edges = np.ascontiguousarray(edges, np.uint32).reshape(-1, 3)
        E = np.zeros((num_nodes, dim), np.float32)
        S = np.zeros((num_nodes, dim), np.float32)
        rE = np.zeros((max(num_rels, 1), dim), np.float32)
        rS = np.zeros((max(num_rels, 1), dim), np.float32)
        loss = np.zeros(1, np.float64)
        et = np.zeros(1, np.uint64)
        bt = np.zeros(1, np.uint64)
        with tempfile.TemporaryDirectory() as d:
            self._check(self._fn["run_epoch_store"](
                os.path.join(d, "s").encode(), _ptr(edges), len(edges), num_nodes, num_rels, n,
                kind, dim, lr, eps, batch_size, k, int(shuffle), seed, epoch, store_seed, _ptr(E),
                _ptr(S), _ptr(rE), _ptr(rS), _ptr(loss), _ptr(et), _ptr(bt)))
        return {"loss_sum": float(loss[0]), "edges_trained": int(et[0]),
                "buckets_trained": int(bt[0]), "E": E, "S": S, "relE": rE[:num_rels],
                "relS": rS[:num_rels]}


def single_state_plan(n):
    """n <= 3: one buffer state holding every partition, buckets row-major
    (the survey's stated n<=3 convention; test_pipeline.cpp:227-269 style)."""
    assert 1 <= n <= 3
    states = np.full((1, 3), 0xFFFFFFFF, np.uint32)
    states[0, :n] = np.arange(n)
    order = np.array([(a, b) for a in range(n) for b in range(n)], np.uint32).reshape(-1, 2)
    return {"n": n, "states": states, "swaps": np.zeros((0, 2), np.uint32),
            "bucket_order": order, "state_offsets": np.array([0, n * n], np.uint64),
            "prefetch_points": np.zeros(0, np.uint64)}
