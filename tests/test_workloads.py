"""Input generators (workloads/): structural contract of every recipe --
simple, symmetric, sorted adjacency, connected, the paper's query protocol."""
import numpy as np
import pytest

import workloads as W


def _check_graph(g):
    d = g.degrees()
    assert g.offsets[0] == 0 and np.all(d > 0)
    rows = np.repeat(np.arange(g.n), d)
    assert not np.any(rows == g.cols)                                  # no self-loops
    key = rows.astype(np.int64) * g.n + g.cols
    assert np.all(np.diff(key) > 0)                                    # sorted rows, no duplicates
    rkey = np.sort(g.cols.astype(np.int64) * g.n + rows)
    assert np.array_equal(rkey, key)                                   # symmetric
    assert W._connected(g)


@pytest.mark.parametrize("scale,ef,abcd", [(12, 5, (0.57, 0.19, 0.19, 0.05)), (11, 16, (0.45, 0.22, 0.22, 0.11))])
def test_rmat_torch_structure(scale, ef, abcd):
    a, b, c, d = abcd
    g = W.rmat_torch(scale, ef, a, b, c, d, seed=7, device="cpu")
    _check_graph(g)
    assert g.n > 0.2 * (1 << scale)
    g2 = W.rmat_torch(scale, ef, a, b, c, d, seed=7, device="cpu")     # seeded: reproducible
    assert np.array_equal(g.offsets, g2.offsets) and np.array_equal(g.cols, g2.cols)


def test_rmat_numpy_and_tiny_structure():
    _check_graph(W.rmat(12, 5, seed=3))
    _check_graph(W.tiny_er())


def test_query_pairs_protocol():
    g = W.rmat(12, 5, seed=3)
    p = W.query_pairs(g, 1001, seed=5)
    assert p.shape == (1001, 2) and p.dtype == np.int32
    half = 1001 // 2
    edges = p[half:]
    adj = set(zip(np.repeat(np.arange(g.n), g.degrees()).tolist(), g.cols.tolist()))
    assert all((int(s), int(t)) in adj for s, t in edges)             # second half: edges
    assert 0.35 < np.mean(edges[:, 0] < edges[:, 1]) < 0.65           # fair-coin orientation
    assert np.array_equal(p, W.query_pairs(g, 1001, seed=5))


def test_rmat_torch_bucketed_dedupe_is_identical():
    """The bucketed torch.unique path (used for billion-arc graphs) builds the same graph."""
    g1 = W.rmat_torch(12, 6, seed=9, device="cpu")
    old = W._UNIQUE_BUCKET
    try:
        W._UNIQUE_BUCKET = 5000
        g2 = W.rmat_torch(12, 6, seed=9, device="cpu")
    finally:
        W._UNIQUE_BUCKET = old
    assert np.array_equal(g1.offsets, g2.offsets) and np.array_equal(g1.cols, g2.cols)
