"""The drop-in boundary: liblegend_b200.so loads, exports every entry point
include/legend_b200.h declares, and refuses to run without a GPU (no CPU
fallback).  CPU only."""
import ctypes
import os
import re

import pytest
from conftest import ROOT

import paper_2505_09258_b200 as lgd
from paper_2505_09258_b200 import legend


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "legend_b200.h")).read()
    return sorted(set(re.findall(r"\b(lgd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(legend.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a():
    blob = open(legend.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lgd.RuntimeFailure):
        lgd.Trainer(lgd.ScoreModel("distmult", 16))
    with pytest.raises(lgd.RuntimeFailure):
        lgd.rng_below(1, 10, 5)


def test_argument_validation_before_device():
    with pytest.raises(lgd.InvalidArgument):
        lgd.Trainer(lgd.ScoreModel("complex", 7))
    with pytest.raises(lgd.InvalidArgument):
        lgd.Trainer(lgd.ScoreModel("dot", 0))
    # shared-negative chunks: dot-product models, dim % 4 == 0 and <= 128 (legend_b200.h)
    for kind, d in (("transe", 64), ("distmult", 130), ("dot", 50)):
        with pytest.raises(lgd.InvalidArgument, match="shared-negative"):
            lgd.Trainer(lgd.ScoreModel(kind, d), lgd.TrainOptions(negatives=8, shared_chunk=64))


def test_store_calls_reject_null_context_without_gpu():
    """The write-back entry points validate before touching a device."""
    L = lgd.library()
    assert L.lgd_store_partition_async(None, 0, None, 0) != 0
    assert b"null" in lgd.library().lgd_last_error()
    assert L.lgd_wait_stores(None) != 0
    assert b"null" in lgd.library().lgd_last_error()
