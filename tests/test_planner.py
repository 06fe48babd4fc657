"""The host planner (paper_2505_09258_b200/csrc/planner.cpp) against the
reference's Algorithms 1-2: identical plans for n = 4..40 (golden vectors from
the reference library), the byte-stable fig6 JSON fixture, and the
structural properties test_ordering.cpp checks.  Host code only: runs on CPU."""
import os

import numpy as np
import pytest
from conftest import GOLDEN, golden

import paper_2505_09258_b200 as lgd

KEYS = ("states", "swaps", "bucket_order", "state_offsets", "prefetch_points")


@pytest.mark.parametrize("n", list(range(4, 41)))
def test_plan_matches_reference(n):
    g = golden("plans")
    p = lgd.plan_iteration_order(n)
    for key in KEYS:
        assert np.array_equal(np.asarray(getattr(p, key)), g[f"n{n}_{key}"]), key


def test_fig6_json_is_byte_identical():
    with open(os.path.join(GOLDEN, "fig6_plan.json")) as f:
        assert lgd.plan_to_json(lgd.plan_iteration_order(6)) == f.read()


def test_published_state_counts():
    # test_ordering.cpp:49-76: this artifact's counts 8 16 24 36 49 68 for n=6..16
    counts = [len(lgd.plan_iteration_order(n).states) for n in (6, 8, 10, 12, 14, 16)]
    assert counts == [8, 16, 24, 36, 49, 68]


@pytest.mark.parametrize("n", [4, 5, 9, 16, 32])
def test_plan_properties(n):
    # test_ordering.cpp:127-172: resident permutation, prefetchable windows
    p = lgd.plan_iteration_order(n)
    order = [tuple(b) for b in p.bucket_order.tolist()]
    assert sorted(order) == [(a, b) for a in range(n) for b in range(n)]
    for s in range(len(p.states)):
        st = set(p.states[s].tolist())
        for g in range(int(p.state_offsets[s]), int(p.state_offsets[s + 1])):
            assert set(order[g]) <= st
    for s in range(len(p.states) - 1):
        ev = int(p.swaps[s][0])
        point, end = int(p.prefetch_points[s]), int(p.state_offsets[s + 1])
        assert point < end  # something to compute while the swap is in flight
        assert all(ev not in order[g] for g in range(point, end))


def test_small_n_rejected():
    with pytest.raises(lgd.InvalidArgument):
        lgd.plan_iteration_order(3)
