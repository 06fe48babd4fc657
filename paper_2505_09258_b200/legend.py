"""Python face of the B200 trainer: a ctypes mirror of the reference trainer's
API (legend::ScoreModel, TrainOptions, run_epoch, batch_loss /
batch_gradients / adagrad_step, sample_negatives, evaluate, the planner and
the E||S store layout) over the C ABI in include/legend_b200.h.

There is no CPU fallback: importing works anywhere, but every compute call
goes through liblegend_b200.so on a CUDA device and raises if the library or
the device is missing.
"""
from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LGD_LIBRARY") or os.path.join(_HERE, "liblegend_b200.so")

MODELS = {"dot": 0, "distmult": 1, "complex": 2, "transe": 3}
NO_RELATION = 0xFFFFFFFF

KSTAT_SCORE, KSTAT_SORT, KSTAT_UPDATE, KSTAT_REL, KSTAT_SAMPLE, KSTAT_SHUFFLE, KSTAT_EVAL = range(7)
KSTAT_NAMES = ["score", "sort", "update", "relations", "sample", "shuffle", "evaluate"]


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference."""


class OutOfRange(IndexError):
    """std::out_of_range in the reference."""


class RuntimeFailure(RuntimeError):
    """std::runtime_error / CUDA failure."""


_ERRORS = {1: InvalidArgument, 2: LogicError, 3: OutOfRange, 4: RuntimeFailure}


class _Options(C.Structure):
    _fields_ = [("learning_rate", C.c_double), ("adagrad_epsilon", C.c_double),
                ("batch_size", C.c_uint32), ("negatives", C.c_uint32), ("shuffle", C.c_int32),
                ("shared_chunk", C.c_uint32), ("seed", C.c_uint64)]


class _EpochResult(C.Structure):
    _fields_ = [("loss_sum", C.c_double), ("loss_per_edge", C.c_double),
                ("edges_trained", C.c_uint64), ("buckets_trained", C.c_uint64),
                ("batches", C.c_uint64), ("wall_seconds", C.c_double),
                ("device_ms", C.c_double), ("unique_nodes", C.c_uint64),
                ("unique_rels", C.c_uint64), ("algorithmic_bytes", C.c_double),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64)]


class _KStats(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("total_ms", C.c_double),
                ("algorithmic_bytes", C.c_double)]


_lib = None


def library():
    """Load liblegend_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeFailure(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                             "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i32, f64 = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
    sig = {
        "lgd_last_error": (C.c_char_p, []),
        "lgd_create": (i32, [vp, i32, u32, vp, i32]),
        "lgd_destroy": (None, [vp]),
        "lgd_set_options": (i32, [vp, vp]),
        "lgd_set_graph": (i32, [vp, vp, u64, u64, u64]),
        "lgd_generate_graph": (i32, [vp, u64, u64, u64, f64, u64]),
        "lgd_get_graph": (i32, [vp, vp]),
        "lgd_make_partition_plan": (i32, [vp, u32, vp, vp]),
        "lgd_set_partition_plan": (i32, [vp, u32, vp, vp]),
        "lgd_plan_iteration_order": (i32, [u32, u64, vp, vp, vp, vp, vp, vp]),
        "lgd_set_iteration_plan": (i32, [vp, u64, vp, vp, vp, vp, vp]),
        "lgd_init_store": (i32, [vp, u64]),
        "lgd_load_partition": (i32, [vp, u32, vp, u64]),
        "lgd_store_partition": (i32, [vp, u32, vp, u64]),
        "lgd_store_partition_async": (i32, [vp, u32, vp, u64]),
        "lgd_wait_stores": (i32, [vp]),
        "lgd_set_relations": (i32, [vp, vp, u64]),
        "lgd_get_relations": (i32, [vp, vp, u64]),
        "lgd_train_epoch": (i32, [vp, u32, vp]),
        "lgd_train_buckets": (i32, [vp, u32, u64, u64, vp]),
        "lgd_train_buckets_from_host": (i32, [vp, u32, u64, u64, vp, vp]),
        "lgd_train_bucket_prefix": (i32, [vp, u32, u64, u64, vp, vp, vp]),
        "lgd_comm_unique_id": (i32, [vp]),
        "lgd_comm_init": (i32, [vp, vp, u32, u32]),
        "lgd_comm_init_local": (i32, [vp, u32]),
        "lgd_round_count": (i32, [vp, vp]),
        "lgd_round_enqueue": (i32, [vp, u32, u32]),
        "lgd_round_handoff": (i32, [vp]),
        "lgd_round_collect": (i32, [vp, vp, vp, vp]),
        "lgd_train_round": (i32, [vp, u32, u32, vp, vp, vp]),
        "lgd_round_actions": (i32, [u32, u32, u32, u32, vp, u64, vp, vp, vp]),
        "lgd_write_graph": (i32, [C.c_char_p, vp, u64, u64, u64]),
        "lgd_read_graph_meta": (i32, [C.c_char_p, vp, vp, vp]),
        "lgd_read_graph": (i32, [C.c_char_p, vp, u64]),
        "lgd_ingest_tsv": (i32, [C.c_char_p, i32, i32, i32, vp, vp, vp, vp]),
        "lgd_free_edges": (None, [vp]),
        "lgd_round_schedule": (i32, [u32, u64, vp, vp, vp, vp]),
        "lgd_train_items": (i32, [vp, u32, vp, u64, vp]),
        "lgd_set_host_edges": (i32, [vp, vp]),
        "lgd_round_begin": (i32, [vp, u32, vp, u64, vp]),
        "lgd_round_step": (i32, [vp, u64, vp]),
        "lgd_round_apply_relations": (i32, [vp, vp]),
        "lgd_round_end": (i32, [vp, vp]),
        "lgd_get_stream": (i32, [vp, vp]),
        "lgd_set_stream_ordered": (i32, [vp, i32]),
        "lgd_device_tables": (i32, [vp, vp, vp, vp, vp]),
        "lgd_get_bucketed_edges": (i32, [vp, vp]),
        "lgd_host_alloc": (i32, [u64, vp]),
        "lgd_host_free": (i32, [vp]),
        "lgd_train_batch": (i32, [vp, vp, u64, vp, i32, vp, vp, vp]),
        "lgd_batch_gradients": (i32, [vp, vp, u64, vp, vp, vp, vp, vp, vp, vp, vp]),
        "lgd_evaluate": (i32, [vp, vp, u64, u32, u32, u64, vp, vp]),
        "lgd_rng_below": (i32, [i32, u64, u64, u64, u64, vp, vp]),
        "lgd_sample_negatives": (i32, [i32, u64, u64, vp, vp, i32, u32, u64, vp, vp]),
        "lgd_shuffle_permutation": (i32, [i32, u64, u64, vp, vp]),
        "lgd_set_profiling": (i32, [vp, i32]),
        "lgd_get_kernel_stats": (i32, [vp, i32, vp]),
        "lgd_reset_kernel_stats": (i32, [vp]),
        "lgd_launch_count": (u64, [vp]),
        "lgd_synchronize": (i32, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc):
    if rc:
        msg = library().lgd_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeFailure)(msg)


def _result(r) -> "EpochResult":
    return EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _u32(a, cols=None):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return a.reshape(-1, cols) if cols else a


# ------------------------------------------------------------ value types
@dataclass
class ScoreModel:
    """ScoreModel (train.hpp:15-23): kind in {"dot", "distmult", "complex"}."""
    kind: str = "dot"
    dim: int = 0

    def uses_relations(self):
        return self.kind != "dot"


@dataclass
class TrainOptions:
    """TrainOptions (pipeline.hpp:89-97) with the reference CLI defaults."""
    learning_rate: float = 0.1
    adagrad_epsilon: float = 1e-10
    batch_size: int = 100000
    negatives: int = 16
    shuffle: bool = True
    seed: int = 0
    # 0: independent negatives per positive (the reference).  C > 0: every C
    # consecutive positives share `negatives` ids (tensor-core scoring; not a
    # reference mode -- DESIGN.md section 4b)
    shared_chunk: int = 0

    def _c(self):
        return _Options(self.learning_rate, self.adagrad_epsilon, self.batch_size,
                        self.negatives, int(self.shuffle), self.shared_chunk, self.seed)

    def batch_negatives(self, positives: int) -> int:
        """Negative ids one batch of `positives` consumes."""
        if self.shared_chunk:
            return -(-positives // self.shared_chunk) * self.negatives
        return positives * self.negatives


@dataclass
class EpochResult:
    """EpochResult (pipeline.hpp:99-107) plus device accounting."""
    loss_sum: float = 0.0
    loss_per_edge: float = 0.0
    edges_trained: int = 0
    buckets_trained: int = 0
    batches: int = 0
    wall_seconds: float = 0.0
    device_ms: float = 0.0
    unique_nodes: int = 0
    unique_rels: int = 0
    algorithmic_bytes: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


@dataclass
class EvalOptions:
    """EvalOptions (train.hpp:123-127)."""
    hits_k: int = 10
    num_candidates: int = 999
    seed: int = 0


@dataclass
class IterationPlan:
    """IterationPlan (ordering.hpp:40-47) as arrays."""
    n: int
    states: np.ndarray
    swaps: np.ndarray
    bucket_order: np.ndarray
    state_offsets: np.ndarray
    prefetch_points: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))

    def as_dict(self):
        return {"n": self.n, "states": self.states, "swaps": self.swaps,
                "bucket_order": self.bucket_order, "state_offsets": self.state_offsets,
                "prefetch_points": self.prefetch_points}


# ---------------------------------------------------------------- planner
def plan_iteration_order(n: int) -> IterationPlan:
    """plan_iteration_order(plan_loading_order(n), n) -- host C++ (n >= 4)."""
    L = library()
    S = np.zeros(1, np.uint64)
    _check(L.lgd_plan_iteration_order(n, 0, _p(S), None, None, None, None, None))
    s = int(S[0])
    states = np.zeros((s, 3), np.uint32)
    swaps = np.zeros((max(s - 1, 1), 2), np.uint32)
    order = np.zeros((n * n, 2), np.uint32)
    soff = np.zeros(s + 1, np.uint64)
    pre = np.zeros(max(s - 1, 1), np.uint64)
    _check(L.lgd_plan_iteration_order(n, s, _p(S), _p(states), _p(swaps), _p(order), _p(soff),
                                      _p(pre)))
    return IterationPlan(n, states, swaps[:s - 1], order, soff, pre[:s - 1])


def single_state_plan(n: int) -> IterationPlan:
    """n <= 3: one buffer state holding every partition, row-major buckets."""
    states = np.full((1, 3), NO_RELATION, np.uint32)
    states[0, :n] = np.arange(n)
    order = np.array([(a, b) for a in range(n) for b in range(n)], np.uint32).reshape(-1, 2)
    return IterationPlan(n, states, np.zeros((0, 2), np.uint32), order,
                         np.array([0, n * n], np.uint64))


def plan_to_json(plan: IterationPlan) -> str:
    """plan_to_json (ordering.cpp:428-440): nlohmann dump(2) canonical text."""
    def arr2(rows, ind):
        if len(rows) == 0:
            return "[]"
        pad, pad2 = " " * ind, " " * (ind + 2)
        inner = []
        for r in rows:
            vals = ",\n".join(pad2 + "  " + str(int(v)) for v in r)
            inner.append(f"{pad2}[\n{vals}\n{pad2}]")
        return "[\n" + ",\n".join(inner) + "\n" + pad + "]"

    def arr1(vals, ind):
        if len(vals) == 0:
            return "[]"
        pad, pad2 = " " * ind, " " * (ind + 2)
        return "[\n" + ",\n".join(pad2 + str(int(v)) for v in vals) + "\n" + pad + "]"

    # nlohmann::json objects are std::map-ordered (keys sorted)
    body = {
        "bucket_order": arr2(plan.bucket_order, 2),
        "loads": arr2(plan.swaps, 2),
        "n": str(int(plan.n)),
        "prefetch_points": arr1(plan.prefetch_points, 2),
        "state_offsets": arr1(plan.state_offsets, 2),
        "states": arr2(plan.states, 2),
    }
    return "{\n" + ",\n".join(f'  "{k}": {v}' for k, v in body.items()) + "\n}\n"


# ------------------------------------------------------ sampler primitives
def rng_below(seed, bound, count, skip=0, device=0):
    """Rng(seed) after `skip` draws: next_below(bound) x count on the device."""
    out = np.zeros(max(count, 1), np.uint64)
    used = np.zeros(1, np.uint64)
    _check(library().lgd_rng_below(device, seed, skip, bound, count, _p(out), _p(used)))
    return out[:count], int(used[0])


def sample_negatives(first, counts, k, num_positives, seed, skip=0, device=0):
    """sample_negatives (train.cpp:365-373) over 1-3 resident node ranges."""
    first = np.ascontiguousarray(first, np.uint64)
    counts = np.ascontiguousarray(counts, np.uint64)
    out = np.zeros(max(num_positives * k, 1), np.uint32)
    used = np.zeros(1, np.uint64)
    _check(library().lgd_sample_negatives(device, seed, skip, _p(first), _p(counts), len(first),
                                          k, num_positives, _p(out), _p(used)))
    return out[:num_positives * k], int(used[0])


def shuffle_permutation(seed, m, device=0):
    """The bucket shuffle of pipeline.cpp:297-301 as a permutation."""
    perm = np.zeros(max(m, 1), np.uint32)
    used = np.zeros(1, np.uint64)
    _check(library().lgd_shuffle_permutation(device, seed, m, _p(perm), _p(used)))
    return perm[:m], int(used[0])


def write_graph(directory, edges, num_nodes, num_relations=0):
    """write_graph (graph.cpp:152-171): edges.bin + graph_meta.json (host only)."""
    edges = _u32(edges, 3)
    _check(library().lgd_write_graph(os.fsencode(directory), _p(edges), len(edges), num_nodes,
                                     num_relations))


def ingest_tsv(path, triples=True, remap_ids=False, threads=0):
    """ingest (graph.cpp:39-118) on host threads: (edges [E x 3] u32, num_nodes,
    num_relations); malformed input raises RuntimeFailure with the line."""
    ptr = C.c_void_p()
    E, V, R = C.c_uint64(), C.c_uint64(), C.c_uint64()
    _check(library().lgd_ingest_tsv(os.fsencode(path), int(triples), int(remap_ids), threads,
                                    C.byref(ptr), C.byref(E), C.byref(V), C.byref(R)))
    try:
        buf = (C.c_uint32 * (3 * E.value)).from_address(ptr.value)
        edges = np.frombuffer(buf, np.uint32).reshape(-1, 3).copy()
    finally:
        library().lgd_free_edges(ptr)
    return edges, V.value, R.value


def read_graph(directory):
    """read_graph (graph.cpp:173-192): (edges [E x 3] u32, num_nodes, num_relations)."""
    E, V, R = C.c_uint64(), C.c_uint64(), C.c_uint64()
    d = os.fsencode(directory)
    _check(library().lgd_read_graph_meta(d, C.byref(E), C.byref(V), C.byref(R)))
    edges = np.zeros((E.value, 3), np.uint32)
    _check(library().lgd_read_graph(d, _p(edges), E.value))
    return edges, V.value, R.value


class _CudaArray:
    """__cuda_array_interface__ shim: wraps a device pointer of f32 values."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PinnedArray:
    """Page-locked host memory (cudaHostAlloc) viewed as a numpy array."""

    def __init__(self, shape, dtype):
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        ptr = C.c_void_p()
        _check(library().lgd_host_alloc(nbytes, C.byref(ptr)))
        self._ptr = ptr
        buf = (C.c_char * max(nbytes, 1)).from_address(ptr.value)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self):
        if getattr(self, "_ptr", None):
            self.array = None
            library().lgd_host_free(self._ptr)
            self._ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ------------------------------------------------------------------ trainer
class Trainer:
    """One HBM-resident training context (graph, partitions, plan, E||S)."""

    def __init__(self, model: ScoreModel, options: TrainOptions | None = None, device: int = 0):
        self.model = model
        self.options = options or TrainOptions()
        self.device = device
        L = library()
        h = C.c_void_p()
        opts = self.options._c()
        _check(L.lgd_create(C.byref(h), MODELS[model.kind], model.dim, C.byref(opts), device))
        self._h = h
        self._ordered = False
        self._stores = []  # host buffers of pending asynchronous write-backs
        self.num_nodes = self.num_relations = self.num_edges = 0
        self.n = 0
        self.bucket_offsets = None

    def close(self):
        if getattr(self, "_h", None):
            library().lgd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_options(self, options: TrainOptions):
        self.options = options
        opts = options._c()
        _check(library().lgd_set_options(self._h, C.byref(opts)))

    # graph -------------------------------------------------------------
    def set_graph(self, edges, num_nodes, num_relations=0):
        edges = _u32(edges, 3)
        _check(library().lgd_set_graph(self._h, _p(edges), len(edges), num_nodes, num_relations))
        self.num_nodes, self.num_relations, self.num_edges = num_nodes, num_relations, len(edges)

    def generate_graph(self, num_nodes, num_relations, num_edges, zipf_exponent=2.1, seed=1):
        _check(library().lgd_generate_graph(self._h, num_nodes, num_relations, num_edges,
                                            zipf_exponent, seed))
        self.num_nodes, self.num_relations, self.num_edges = num_nodes, num_relations, num_edges

    def get_graph(self):
        out = np.zeros((self.num_edges, 3), np.uint32)
        _check(library().lgd_get_graph(self._h, _p(out)))
        return out

    def make_partition_plan(self, n, want_edge_order=False):
        offsets = np.zeros(n * n + 1, np.uint64)
        order = np.zeros(max(self.num_edges, 1), np.uint64) if want_edge_order else None
        _check(library().lgd_make_partition_plan(self._h, n, _p(offsets), _p(order)))
        self.n, self.bucket_offsets = n, offsets
        return offsets, (order[:self.num_edges] if order is not None else None)

    def set_partition_plan(self, n, bucket_offsets, edge_order):
        bucket_offsets = np.ascontiguousarray(bucket_offsets, np.uint64)
        edge_order = np.ascontiguousarray(edge_order, np.uint64)
        _check(library().lgd_set_partition_plan(self._h, n, _p(bucket_offsets), _p(edge_order)))
        self.n, self.bucket_offsets = n, bucket_offsets

    def set_iteration_plan(self, plan):
        if isinstance(plan, dict):
            plan = IterationPlan(**{k: plan[k] for k in ("n", "states", "swaps", "bucket_order",
                                                         "state_offsets")},
                                 prefetch_points=plan.get("prefetch_points",
                                                          np.zeros(0, np.uint64)))
        st = _u32(plan.states, 3)
        sw = _u32(plan.swaps, 2) if len(plan.swaps) else None
        bo = _u32(plan.bucket_order, 2)
        so = np.ascontiguousarray(plan.state_offsets, np.uint64)
        pp = np.ascontiguousarray(plan.prefetch_points, np.uint64) if len(
            plan.prefetch_points) else None
        _check(library().lgd_set_iteration_plan(self._h, len(st), _p(st), _p(sw), _p(bo), _p(so),
                                                _p(pp)))

    # store ---------------------------------------------------------------
    def stride(self):
        return (self.num_nodes + self.n - 1) // self.n

    def part_rows(self, p):
        s = self.stride()
        return max(0, min(s * (p + 1), self.num_nodes) - s * p)

    def init_store(self, seed):
        """EmbeddingStore::create initial values (store.cpp:59-86) on the device."""
        _check(library().lgd_init_store(self._h, seed))

    def load_partition(self, p, e_s):
        e_s = np.ascontiguousarray(e_s, np.float32)
        _check(library().lgd_load_partition(self._h, p, _p(e_s), self.part_rows(p)))

    def store_partition(self, p):
        rows = self.part_rows(p)
        out = np.zeros(2 * rows * self.model.dim, np.float32)
        _check(library().lgd_store_partition(self._h, p, _p(out), rows))
        return out

    def store_partition_async(self, p, out):
        """Queue the write-back of partition p into `out` (a float32 array of
        2 * rows * dim, ideally PinnedArray.array) and return at once; the copy
        overlaps later read-only work (evaluate).  `out` is filled when
        wait_stores() returns (EmbeddingStore::write_partition, store.cpp:27-57)."""
        rows = self.part_rows(p)
        if not (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
                and out.size == 2 * rows * self.model.dim):
            raise ValueError("out must be a contiguous float32 array of 2 * rows * dim")
        _check(library().lgd_store_partition_async(self._h, p, _p(out), rows))
        self._stores.append(out)

    def wait_stores(self):
        _check(library().lgd_wait_stores(self._h))
        self._stores.clear()

    def load_tables(self, E, S):
        """Whole-graph E and S (V x d) split into the n E||S partition blobs."""
        s = self.stride()
        for p in range(self.n):
            a, b = s * p, min(s * (p + 1), self.num_nodes)
            self.load_partition(p, np.concatenate([E[a:b].ravel(), S[a:b].ravel()]))

    def tables(self):
        """(E, S) as whole-graph V x d arrays."""
        d = self.model.dim
        E = np.zeros((self.num_nodes, d), np.float32)
        S = np.zeros((self.num_nodes, d), np.float32)
        s = self.stride()
        for p in range(self.n):
            a, b = s * p, min(s * (p + 1), self.num_nodes)
            blob = self.store_partition(p)
            E[a:b] = blob[:(b - a) * d].reshape(-1, d)
            S[a:b] = blob[(b - a) * d:].reshape(-1, d)
        return E, S

    def set_relations(self, relE, relS):
        blob = np.concatenate([np.ravel(relE), np.ravel(relS)]).astype(np.float32)
        _check(library().lgd_set_relations(self._h, _p(blob), self.num_relations))

    def get_relations(self):
        d = self.model.dim
        blob = np.zeros(max(2 * self.num_relations * d, 1), np.float32)
        _check(library().lgd_get_relations(self._h, _p(blob), self.num_relations))
        r = self.num_relations * d
        return blob[:r].reshape(-1, d), blob[r:2 * r].reshape(-1, d)

    # training ----------------------------------------------------------
    def run_epoch(self, epoch=0) -> EpochResult:
        """run_epoch real-train (pipeline.cpp:273-322) over the HBM-resident table."""
        r = _EpochResult()
        _check(library().lgd_train_epoch(self._h, epoch, C.byref(r)))
        return EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})

    def train_buckets(self, epoch, g_begin, g_end) -> EpochResult:
        r = _EpochResult()
        _check(library().lgd_train_buckets(self._h, epoch, g_begin, g_end, C.byref(r)))
        return EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})

    def train_bucket_prefix(self, epoch, g, max_batches=0):
        """The bucket at plan position g, cut after max_batches batches (0 =
        all): returns (EpochResult, per-batch losses, per-batch unique nodes)."""
        sizes = np.diff(np.asarray(self.bucket_offsets, np.int64))
        cap = int(-(-sizes.max() // self.options.batch_size)) if len(sizes) else 0
        if max_batches:
            cap = min(cap, max_batches)
        losses = np.zeros(max(cap, 1), np.float64)
        nodes = np.zeros(max(cap, 1), np.uint64)
        r = _EpochResult()
        _check(library().lgd_train_bucket_prefix(self._h, epoch, g, max_batches, _p(losses),
                                                 _p(nodes), C.byref(r)))
        res = EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})
        return res, losses[:res.batches], nodes[:res.batches]

    def train_buckets_from_host(self, epoch, g_begin, g_end, host_bucketed) -> EpochResult:
        """train_buckets with each bucket's edges copied H2D from host memory."""
        r = _EpochResult()
        _check(library().lgd_train_buckets_from_host(self._h, epoch, g_begin, g_end,
                                                     _p(host_bucketed), C.byref(r)))
        return EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})

    def set_host_edges(self, host_bucketed=None):
        """Stream every bucket H2D from this host copy of the bucket-ordered
        edges (None: back to the device-resident copy); keep it alive."""
        self._host_edges = host_bucketed
        _check(library().lgd_set_host_edges(self._h, _p(host_bucketed) if host_bucketed is not None
                                            else None))

    def bucketed_edges(self, out=None):
        """The edge list in bucket order (into `out`, e.g. a PinnedArray view)."""
        if out is None:
            out = np.zeros((self.num_edges, 3), np.uint32)
        _check(library().lgd_get_bucketed_edges(self._h, _p(out)))
        return out

    # ---- multi-GPU round schedule (paper_2505_09258_b200/multigpu.py) ------
    @property
    def typed(self):
        return self.model.uses_relations()

    def train_items(self, epoch, items) -> EpochResult:
        """Train an explicit bucket list (structured lgd_bucket_item array)."""
        items = np.ascontiguousarray(items)
        r = _EpochResult()
        _check(library().lgd_train_items(self._h, epoch, items.ctypes.data_as(C.c_void_p),
                                         len(items), C.byref(r)))
        return EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})

    def round_begin(self, epoch, items) -> int:
        items = np.ascontiguousarray(items)
        self._round_items = items  # keep alive
        nb = np.zeros(1, np.uint64)
        _check(library().lgd_round_begin(self._h, epoch, items.ctypes.data_as(C.c_void_p),
                                         len(items), _p(nb)))
        return int(nb[0])

    def round_step(self, step, rel_buf):
        """rel_buf: device tensor [R x (d+1)] f64 (torch) or None."""
        ptr = None if rel_buf is None else C.c_void_p(rel_buf.data_ptr())
        _check(library().lgd_round_step(self._h, step, ptr))

    def round_apply(self, summed):
        """One relation Adagrad step from the summed [R x (d+1)] buffer.  The
        trainer runs on its own CUDA stream: work torch queued on `summed`
        (the NCCL all-reduce, a sum) is finished first -- by the stream order
        itself in stream-ordered mode (see stream_ordered), else by draining
        torch's current stream."""
        if getattr(summed, "is_cuda", False) and not self._ordered:
            import torch
            torch.cuda.current_stream(summed.device).synchronize()
        _check(library().lgd_round_apply_relations(self._h, C.c_void_p(summed.data_ptr())))

    def cuda_stream(self):
        """The trainer's CUDA stream as a torch.cuda.ExternalStream."""
        import torch
        ptr = C.c_void_p()
        _check(library().lgd_get_stream(self._h, C.byref(ptr)))
        return torch.cuda.ExternalStream(ptr.value or 0, device=f"cuda:{self.device}")

    @contextlib.contextmanager
    def stream_ordered(self):
        """Lock-step rounds without host round trips: inside the block,
        round_step / round_apply only queue work on the trainer's stream, which
        is torch's current stream, so a collective issued between them (NCCL
        orders itself after the current stream and makes it wait for the
        result) runs in stream order.  The stream is drained on exit."""
        import torch
        st = self.cuda_stream()
        self.set_stream_ordered(True)
        try:
            with torch.cuda.stream(st):
                yield st
        finally:
            self.set_stream_ordered(False)
            st.synchronize()

    def set_stream_ordered(self, on: bool):
        """lgd_set_stream_ordered; prefer the stream_ordered() block."""
        _check(library().lgd_set_stream_ordered(self._h, int(bool(on))))
        self._ordered = bool(on)

    def round_end(self) -> EpochResult:
        r = _EpochResult()
        _check(library().lgd_round_end(self._h, C.byref(r)))
        return EpochResult(**{f: getattr(r, f) for f, _ in _EpochResult._fields_})

    def device_tables(self):
        ptrs = [C.c_void_p() for _ in range(4)]
        _check(library().lgd_device_tables(self._h, *[C.byref(x) for x in ptrs]))
        return [x.value for x in ptrs]

    def partition_views(self, p):
        """Zero-copy torch views (CUDA) of partition p's theta and state rows.
        Trainer calls return with their stream drained; work torch queues on
        these views (NCCL send / recv, copies) must be finished before the
        next trainer call (multigpu.py synchronises after each exchange)."""
        import torch
        th, st, _, _ = self.device_tables()
        s = self.stride()
        a, b = s * p, min(s * (p + 1), self.num_nodes)
        d = self.model.dim
        return [torch.as_tensor(_CudaArray(ptr + a * d * 4, ((b - a) * d,)),
                                device=f"cuda:{self.device}")
                for ptr in (th, st)]

    def train_batch(self, edges, negatives, apply=True):
        """batch_loss + batch_gradients + adagrad_step on one batch."""
        edges = _u32(edges, 3)
        negs = _u32(negatives)
        loss = np.zeros(1, np.float64)
        nn = np.zeros(1, np.uint64)
        nr = np.zeros(1, np.uint64)
        _check(library().lgd_train_batch(self._h, _p(edges), len(edges), _p(negs), int(apply),
                                         _p(loss), _p(nn), _p(nr)))
        return {"loss": float(loss[0]), "nodes": int(nn[0]), "rels": int(nr[0])}

    def batch_gradients(self, edges, negatives):
        """batch_gradients (train.cpp:280-340): sorted ids + FP64 rows."""
        edges = _u32(edges, 3)
        negs = _u32(negatives)
        P, k, d = len(edges), self.options.negatives, self.model.dim
        loss = np.zeros(1, np.float64)
        nn = np.zeros(1, np.uint64)
        nr = np.zeros(1, np.uint64)
        cap = min(P * (k + 2), max(self.num_nodes, 1)) + 1
        ids = np.zeros(cap, np.uint32)
        g = np.zeros((cap, d), np.float64)
        rids = np.zeros(P + 1, np.uint32)
        rg = np.zeros((P + 1, d), np.float64)
        _check(library().lgd_batch_gradients(self._h, _p(edges), P, _p(negs), _p(loss), _p(nn),
                                             _p(ids), _p(g), _p(nr), _p(rids), _p(rg)))
        a, b = int(nn[0]), int(nr[0])
        return {"loss": float(loss[0]), "node_ids": ids[:a], "node_grads": g[:a],
                "rel_ids": rids[:b], "rel_grads": rg[:b]}

    def evaluate(self, test_edges, options: EvalOptions | None = None):
        """evaluate (train.cpp:375-412): (mrr, hits@k)."""
        o = options or EvalOptions()
        test_edges = _u32(test_edges, 3)
        mrr = np.zeros(1, np.float64)
        hits = np.zeros(1, np.float64)
        _check(library().lgd_evaluate(self._h, _p(test_edges), len(test_edges), o.num_candidates,
                                      o.hits_k, o.seed, _p(mrr), _p(hits)))
        return float(mrr[0]), float(hits[0])

    # profiling -----------------------------------------------------------
    def set_profiling(self, on=True):
        _check(library().lgd_set_profiling(self._h, int(on)))

    def kernel_stats(self):
        out = {}
        for i, name in enumerate(KSTAT_NAMES):
            s = _KStats()
            _check(library().lgd_get_kernel_stats(self._h, i, C.byref(s)))
            out[name] = {"launches": s.launches, "total_ms": s.total_ms,
                         "algorithmic_bytes": s.algorithmic_bytes}
        return out

    def reset_kernel_stats(self):
        _check(library().lgd_reset_kernel_stats(self._h))

    def launch_count(self):
        return int(library().lgd_launch_count(self._h))

    def synchronize(self):
        _check(library().lgd_synchronize(self._h))
