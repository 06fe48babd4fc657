"""The device power-law generator (lgd_generate_graph, graph.cu) against its
host restatement (oracle/graphgen.c), edge for edge, at the BASELINE shapes'
node and relation counts; and a generated graph through the reference file
format (lgd_write_graph / lgd_read_graph).  Runs on a B200 (-m gpu)."""
import numpy as np
import pytest

import paper_2505_09258_b200 as lgd

pytestmark = pytest.mark.gpu
ALPHA, SEED = 2.3, 20250509


@pytest.mark.parametrize("V,R", [(15_000, 1345), (4_800_000, 0), (41_600_000, 16),
                                 (86_000_000, 14_800), (65_000_000, 1)])
def test_device_generator_matches_host_restatement(oracle, V, R):
    E = 4_000_000
    t = lgd.Trainer(lgd.ScoreModel("distmult" if R else "dot", 8))
    try:
        t.generate_graph(V, R, E, ALPHA, SEED)
        got = t.get_graph()
    finally:
        t.close()
    want = oracle.powerlaw_edges(V, R, ALPHA, SEED, 0, E)
    bad = np.flatnonzero((got != want).any(1))
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])


def test_generated_graph_file_round_trip(tmp_path, oracle):
    t = lgd.Trainer(lgd.ScoreModel("distmult", 8))
    try:
        t.generate_graph(100_000, 16, 500_000, ALPHA, SEED)
        edges = t.get_graph()
    finally:
        t.close()
    lgd.write_graph(tmp_path / "g", edges, 100_000, 16)
    back, V, R = lgd.read_graph(tmp_path / "g")
    assert (V, R) == (100_000, 16) and np.array_equal(back, edges)
    assert np.array_equal(edges, oracle.powerlaw_edges(100_000, 16, ALPHA, SEED, 0, 500_000))
