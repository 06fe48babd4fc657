"""B200-native partitioned graph-embedding training (Legend, arXiv 2505.09258).

Hot path: hand-written sm_100a CUDA in liblegend_b200.so behind the C ABI of
include/legend_b200.h; this package is the thin Python face of that ABI.
"""
from .legend import (EpochResult, EvalOptions, InvalidArgument, IterationPlan, LogicError,
                     OutOfRange, PinnedArray, RuntimeFailure, ScoreModel, Trainer, TrainOptions, library,
                     ingest_tsv, plan_iteration_order, plan_to_json, read_graph, rng_below, sample_negatives,
                     shuffle_permutation, single_state_plan, write_graph)

__all__ = ["EpochResult", "EvalOptions", "InvalidArgument", "IterationPlan", "LogicError",
           "OutOfRange", "PinnedArray", "RuntimeFailure", "ScoreModel", "Trainer", "TrainOptions", "library",
           "ingest_tsv", "plan_iteration_order", "plan_to_json", "read_graph", "rng_below", "sample_negatives",
           "shuffle_permutation", "single_state_plan", "write_graph"]
