"""Graph format and the synthetic generator, on the CPU.

* lgd_write_graph / lgd_read_graph against the reference's own write_graph /
  read_graph (graph.cpp:152-192): files written by either side are read by the
  other, and graph_meta.json is byte-identical.
* lgd_ingest_tsv against the reference's ingest (graph.cpp:39-118): the same
  edges, counts and remapped ids, and the same ParseError text with the line
  number, for files parsed by several host threads.
* The host restatement of the power-law generator (oracle/graphgen.c, the
  workload of bench.py's reference arm): determinism, counter-based chunking,
  bucket extraction, and its degree distribution.  tests/test_gpu_graph.py
  checks the device generator against it edge for edge.
"""
import os

import numpy as np
import pytest

import paper_2505_09258_b200 as lgd

ALPHA, SEED = 2.3, 20250509


def _random_graph(rng, V=1000, R=7, E=5000, typed=True):
    return np.stack([rng.integers(0, V, E),
                     rng.integers(0, R, E) if typed else np.full(E, 0xFFFFFFFF),
                     rng.integers(0, V, E)], 1).astype(np.uint32)


@pytest.mark.parametrize("typed", [True, False])
def test_write_graph_read_by_reference(tmp_path, reference, typed):
    edges = _random_graph(np.random.default_rng(1), typed=typed)
    lgd.write_graph(tmp_path / "g", edges, 1000, 7 if typed else 0)
    got, V, R = reference.read_graph(tmp_path / "g")
    assert (V, R) == (1000, 7 if typed else 0)
    assert np.array_equal(got, edges)


def test_reference_graph_read_by_lgd_and_meta_bytes(tmp_path, reference):
    edges = _random_graph(np.random.default_rng(2))
    reference.write_graph(tmp_path / "ref", edges, 1000, 7)
    got, V, R = lgd.read_graph(tmp_path / "ref")
    assert (V, R) == (1000, 7) and np.array_equal(got, edges)
    lgd.write_graph(tmp_path / "ours", edges, 1000, 7)
    for name in ("graph_meta.json", "edges.bin"):
        a = open(tmp_path / "ref" / name, "rb").read()
        b = open(tmp_path / "ours" / name, "rb").read()
        assert a == b, name


def test_empty_graph_round_trip(tmp_path):
    lgd.write_graph(tmp_path / "e", np.zeros((0, 3), np.uint32), 5, 0)
    edges, V, R = lgd.read_graph(tmp_path / "e")
    assert edges.shape == (0, 3) and (V, R) == (5, 0)


def test_read_graph_errors(tmp_path):
    with pytest.raises(lgd.RuntimeFailure, match="missing graph_meta.json"):
        lgd.read_graph(tmp_path / "nothing")
    edges = _random_graph(np.random.default_rng(3), E=10)
    lgd.write_graph(tmp_path / "t", edges, 1000, 7)
    with open(tmp_path / "t" / "edges.bin", "r+b") as f:  # truncate: test_graph_store.cpp:244-246
        f.truncate(12 * 9 + 5)
    with pytest.raises(lgd.RuntimeFailure, match="shorter than metadata"):
        lgd.read_graph(tmp_path / "t")


def test_generator_is_counter_based_and_deterministic(oracle):
    V, R = 41_600_000, 16
    whole = oracle.powerlaw_edges(V, R, ALPHA, SEED, 0, 20_000)
    again = oracle.powerlaw_edges(V, R, ALPHA, SEED, 0, 20_000)
    parts = np.concatenate([oracle.powerlaw_edges(V, R, ALPHA, SEED, a, a + 5000)
                            for a in range(0, 20_000, 5000)])
    assert np.array_equal(whole, again) and np.array_equal(whole, parts)
    other = oracle.powerlaw_edges(V, R, ALPHA, SEED + 1, 0, 20_000)
    assert (other != whole).any()
    assert whole[:, [0, 2]].max() < V and whole[:, 1].max() < R
    untyped = oracle.powerlaw_edges(V, 0, ALPHA, SEED, 0, 100)
    assert (untyped[:, 1] == 0xFFFFFFFF).all()
    assert np.array_equal(untyped[:, [0, 2]], whole[:100, [0, 2]])


def test_det_pow_accuracy(oracle):
    rng = np.random.default_rng(5)
    for x, y in zip(1.0 + rng.random(2000) * 1e6, rng.random(2000) * 6):
        got = oracle._fn["det_pow"](float(x), float(y))
        assert abs(got / x ** y - 1) < 1e-13
    assert oracle._fn["det_pow"](1.0, 4.3) == 1.0


@pytest.mark.parametrize("n,bi,bj", [(4, 0, 1), (4, 3, 3), (16, 0, 1)])
def test_bucket_extraction_matches_filter(oracle, n, bi, bj):
    V, R, E = 200_000, 16, 300_000
    edges = oracle.powerlaw_edges(V, R, ALPHA, SEED, 0, E)
    stride = -(-V // n)
    want = edges[(edges[:, 0] // stride == bi) & (edges[:, 2] // stride == bj)]
    for threads in (1, 7):
        got = oracle.powerlaw_bucket(V, R, E, ALPHA, SEED, n, bi, bj, threads=threads)
        assert np.array_equal(got, want)


def test_degree_distribution_is_power_law(oracle):
    """Zipf ranks with density ~ x^-beta, beta = 1/(alpha-1): the degree of
    the rank-r node falls as r^-beta, the top node holds ~0.3% of endpoints
    at Twitter's size (its largest in-degree share is ~0.2%), and hubs are
    scattered over every partition by the multiplicative permutation."""
    V, E = 41_600_000, 2_000_000
    edges = oracle.powerlaw_edges(V, 0, ALPHA, SEED, 0, E)
    ends = np.concatenate([edges[:, 0], edges[:, 2]]).astype(np.int64)
    deg = np.bincount(ends, minlength=V)
    top = np.sort(deg)[::-1]
    share = top[0] / len(ends)
    assert 0.002 < share < 0.005, share
    beta = 1.0 / (ALPHA - 1.0)
    r = np.arange(1, 1001)
    slope = np.polyfit(np.log(r[9:]), np.log(top[9:1000]), 1)[0]
    assert abs(slope + beta) < 0.08, slope
    # the 100 largest hubs land in many of the 16 partitions
    hubs = np.argsort(deg)[::-1][:100]
    assert len(np.unique(hubs // -(-V // 16))) >= 12


def _tsv(rng, n, triples, sparse=False, junk=True):
    lines = ["# a comment line"]
    hi = 10**12 if sparse else 5000
    for i in range(n):
        cols = [rng.integers(0, hi)] + ([rng.integers(0, 40)] if triples else []) + \
               [rng.integers(0, hi)]
        sep = "\t" if i % 3 else "  \t "
        lines.append(sep.join(str(c) for c in cols) + ("\r" if i % 7 == 0 else ""))
        if junk and i % 50 == 0:
            lines += ["", "   ", "#x 1 2"]
    return "\n".join(lines) + ("\n" if n % 2 else "")


@pytest.mark.parametrize("triples", [True, False])
@pytest.mark.parametrize("remap", [False, True])
@pytest.mark.parametrize("threads", [1, 5])
def test_ingest_matches_reference(tmp_path, reference, triples, remap, threads):
    rng = np.random.default_rng(4)
    path = tmp_path / "edges.tsv"
    path.write_text(_tsv(rng, 20000, triples, sparse=remap))
    want = reference.ingest(path, triples, remap)
    got = lgd.ingest_tsv(path, triples, remap, threads=threads)
    assert got[1:] == want[1:]
    assert np.array_equal(got[0], want[0])


@pytest.mark.parametrize("text,msg", [
    ("1 2 3\n4 5\n", "line 2: expected 3 columns, got 2"),
    ("1 2 3\n# c\n\n7 x 9\n", "line 4: malformed integer field 'x'"),
    ("1 2 3\n4 -5 6\n", "line 2: malformed integer field '-5'"),
    ("# only comments\n\n", "edge file has no edges"),
])
def test_ingest_errors_match_reference(tmp_path, reference, text, msg):
    path = tmp_path / "bad.tsv"
    path.write_text(text)
    with pytest.raises(lgd.RuntimeFailure, match=msg):
        lgd.ingest_tsv(path, True, False, threads=3)
    with pytest.raises(Exception, match=msg):
        reference.ingest(path, True, False)


def test_ingest_large_file_parallel(tmp_path, reference):
    rng = np.random.default_rng(9)
    path = tmp_path / "big.tsv"
    edges = np.stack([rng.integers(0, 10**6, 400000), rng.integers(0, 100, 400000),
                      rng.integers(0, 10**6, 400000)], 1)
    np.savetxt(path, edges, fmt="%d", delimiter="\t")
    got = lgd.ingest_tsv(path, True, False, threads=8)
    assert np.array_equal(got[0], edges.astype(np.uint32))
    assert got[1:] == (int(edges[:, [0, 2]].max()) + 1, int(edges[:, 1].max()) + 1)
    assert np.array_equal(reference.ingest(path)[0], got[0])


def test_ingest_error_line_in_a_later_chunk(tmp_path, reference):
    rng = np.random.default_rng(10)
    text = _tsv(rng, 30000, True).split("\n")
    text[25001] = "1 2"  # deep in the file: another thread's chunk
    path = tmp_path / "late.tsv"
    path.write_text("\n".join(text))
    with pytest.raises(Exception) as ref_err:
        reference.ingest(path)
    with pytest.raises(lgd.RuntimeFailure) as err:
        lgd.ingest_tsv(path, True, False, threads=7)
    assert str(err.value) == str(ref_err.value).split(": ", 1)[1] or \
        str(err.value) in str(ref_err.value)
    assert "line 25002: expected 3 columns, got 2" in str(err.value)
