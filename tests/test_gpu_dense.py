"""GPU parity of the SMM head's dense mode (R25) and of K9's exact
summation order.

The dense mode applies an SMM iteration as a pull over the whole CSR (K9) instead of the sparse
push (K2/K3).  It is a schedule of the same arithmetic: every output bit (estimates and all
per-query stats) equals the frontier mode's, and the oracle's (tests/test_gpu_parity.py's
acceptance), on every graph with sorted adjacency lists -- hubs included, because the dense
mode's K9 sums every row sequentially in CSR order (ER_SPMM_EXACT).
"""
import numpy as np
import pytest

import oracle
import workloads as W
from oracle import exact

from test_gpu_parity import _hub_graph, compare, run_both

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("q", [1, 2, 7, 64, 256])
def test_spmm_k9_exact_every_row(geer, q):
    """ER_SPMM_EXACT: every row, hubs of degree 2999 and 1500 included, bit-identical to the
    oracle's sequential dense pull (R13), for A and P = D^-1 A."""
    import torch
    g = _hub_graph()
    d = g.degrees()
    assert (d > 512).sum() >= 2
    h = geer.er_graph_create(g.n, g.offsets, g.cols, flags=geer.ER_CREATE_SPMM_ONLY)
    try:
        X = np.random.default_rng(100 + q).random((g.n, q))
        Xd = torch.from_numpy(X).cuda()
        for normalize in (True, False):
            Y = torch.full((g.n, q), np.nan, dtype=torch.float64, device="cuda")
            geer.er_spmm(h, Xd, Y, normalize=normalize, exact=True)
            Yh = Y.cpu().numpy()
            for c in range(q) if q <= 8 else (0, 1, q // 2, q - 1):
                want = oracle.propagate_dense(g, X[:, c], normalize=normalize)
                assert np.array_equal(Yh[:, c], want), (q, c, normalize)
    finally:
        geer.er_graph_destroy(h)


def test_spmm_ex_rejects_unknown_flags(geer):
    import ctypes
    import torch
    g = _hub_graph(800, 3)
    h = geer.er_graph_create(g.n, g.offsets, g.cols, flags=geer.ER_CREATE_SPMM_ONLY)
    try:
        X = torch.zeros((g.n, 2), dtype=torch.float64, device="cuda")
        Y = torch.zeros_like(X)
        rc = geer.lib.er_spmm_ex(h, ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Y.data_ptr()), 2, 4, None)
        assert rc == geer.ER_EINVAL and "flags" in geer.er_last_error_message()
    finally:
        geer.er_graph_destroy(h)


def _modes(geer, h, pairs, eps, **kw):
    """(r, stats, dense waves) for smm_mode = frontier, dense, auto."""
    out = {}
    for mode in (geer.SMM_FRONTIER, geer.SMM_DENSE, geer.SMM_AUTO):
        geer.er_graph_profile(h, True)
        r, st = geer.er_query_batch_ex(h, pairs, eps, 0.01, stats=True, smm_mode=mode, **kw)
        p = geer.er_graph_profile_read(h)
        geer.er_graph_profile(h, False)
        out[mode] = (r, st, p["smm_dense_waves"], p["smm_waves"])
    return out


def _assert_identical(geer, out):
    r1, s1, d1, w1 = out[geer.SMM_FRONTIER]
    r2, s2, d2, w2 = out[geer.SMM_DENSE]
    r0, s0, _, _ = out[geer.SMM_AUTO]
    assert d1 == 0
    assert d2 == w2 and w2 == w1, (d2, w2, w1)   # every wave after the first ran dense
    assert r2.tobytes() == r1.tobytes() and s2.tobytes() == s1.tobytes()
    assert r0.tobytes() == r1.tobytes() and s0.tobytes() == s1.tobytes()


@pytest.mark.parametrize("eps,kw", [(0.5, {}), (0.1, {}), (0.05, {}), (0.1, dict(force_ell_b=4))])
def test_tiny_dense_mode_parity(geer, tiny, eps, kw):
    g, pairs = tiny
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        geer.er_graph_set_lambda(h, g.lam)
        out = _modes(geer, h, pairs, eps, **kw)
        _assert_identical(geer, out)
        if kw:
            assert out[geer.SMM_DENSE][3] > 0
        r, st, ro, so = run_both(geer, h, g, pairs, eps, smm_mode=geer.SMM_DENSE, **kw)
        compare(g, pairs, r, st, ro, so)
    finally:
        geer.er_graph_destroy(h)


def test_hub_graph_dense_mode_parity(geer):
    """Queries at and around the hubs (rows cut into K9 segments by the non-exact order): the
    dense mode stays bit-identical to the push and to the oracle."""
    g = _hub_graph()
    g.lam = exact.lambda_dense(g)   # the dense eigensolver's lambda on both sides (R12)
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        geer.er_graph_set_lambda(h, g.lam)
        rng = np.random.default_rng(11)
        pairs = np.stack([np.r_[0, 1, 2, 3, rng.integers(0, g.n, 60)],
                          np.r_[1, 5, 3, 700, rng.integers(0, g.n, 60)]], axis=1).astype(np.int32)
        for eps in (0.2, 0.05):
            out = _modes(geer, h, pairs, eps, force_ell_b=4)
            _assert_identical(geer, out)
            assert out[geer.SMM_DENSE][3] > 0
            r, st, ro, so = run_both(geer, h, g, pairs, eps, force_ell_b=4, smm_mode=geer.SMM_DENSE)
            compare(g, pairs, r, st, ro, so)
    finally:
        geer.er_graph_destroy(h)


def test_rmat20_dense_mode_byte_identical(geer, rmat20):
    """BASELINE config 1's graph: 120 queries (every wave fits the dense limit) at eps = 0.05
    (the heaviest SMM heads): dense, push and the cost model give the same bits; the oracle
    agrees on a sample."""
    g, pairs, _, h = rmat20
    sub = np.ascontiguousarray(pairs[:120])
    out = _modes(geer, h, sub, 0.05)
    _assert_identical(geer, out)
    r, st, ro, so = run_both(geer, h, g, sub[:20], 0.05, smm_mode=geer.SMM_DENSE)
    compare(g, sub[:20], r, st, ro, so)


def test_rmat20_cost_model_picks_dense_for_dense_supports(geer, rmat20):
    """Few queries forced through 6 SMM iterations: their supports cover much of the graph, so
    the push would emit ~10^7 pairs per wave and the cost model takes the dense pull (same
    bits)."""
    g, pairs, _, h = rmat20
    sub = np.ascontiguousarray(pairs[:8])
    out = _modes(geer, h, sub, 0.05, force_ell_b=6)
    r1, s1, _, w1 = out[geer.SMM_FRONTIER]
    r0, s0, d0, w0 = out[geer.SMM_AUTO]
    assert w0 == w1 and 0 < d0 <= w0
    assert r0.tobytes() == r1.tobytes() and s0.tobytes() == s1.tobytes()


def test_unsorted_rows_dense_mode_matches_oracle_order(geer, tiny):
    """Adjacency rows in random order: the push sums in ascending source order (within 1e-10 of
    the oracle, R13) but the dense pull sums in CSR order -- the oracle's order -- so with
    smm_mode = dense r_b and psi are bit-identical to the oracle even here."""
    g0, pairs = tiny
    rng = np.random.default_rng(9)
    cols = g0.cols.copy()
    for v in range(g0.n):
        a, b = g0.offsets[v], g0.offsets[v + 1]
        cols[a:b] = rng.permutation(cols[a:b])
    g = W.Graph(g0.n, g0.offsets.copy(), cols, "tiny_shuffled", g0.lam)
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        geer.er_graph_set_lambda(h, g.lam)
        for kw in ({}, dict(force_ell_b=4)):
            r, st, ro, so = run_both(geer, h, g, pairs, 0.1, smm_mode=geer.SMM_DENSE, **kw)
            compare(g, pairs, r, st, ro, so, sorted_adj=True)
            r1, st1, _, _ = run_both(geer, h, g, pairs, 0.1, smm_mode=geer.SMM_FRONTIER, **kw)
            compare(g, pairs, r1, st1, ro, so, sorted_adj=False)
    finally:
        geer.er_graph_destroy(h)


def test_unsorted_rows_bits_do_not_depend_on_batch(geer, tiny):
    """Shuffled adjacency rows: with the default smm_mode (cost model), a query's bits must not
    depend on the other queries of its batch (dist.py's sharding claim).  The automatic dense
    switch is off on unsorted rows (the pull would sum in CSR order, the push in ascending source
    order), so each query run alone -- where the cost model would otherwise pick the pull --
    gives the bits it gets inside the whole batch."""
    g0, pairs = tiny
    rng = np.random.default_rng(19)
    cols = g0.cols.copy()
    for v in range(g0.n):
        a, b = g0.offsets[v], g0.offsets[v + 1]
        cols[a:b] = rng.permutation(cols[a:b])
    g = W.Graph(g0.n, g0.offsets.copy(), cols, "tiny_shuffled", g0.lam)
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        geer.er_graph_set_lambda(h, g.lam)
        for kw in (dict(force_ell_b=4), dict(force_ell_b=6)):
            rall, sall = geer.er_query_batch_ex(h, pairs, 0.05, 0.01, stats=True, **kw)
            for i in range(0, len(pairs), 9):
                r1, s1 = geer.er_query_batch_ex(h, pairs[i:i + 1], 0.05, 0.01, stats=True,
                                                query_ids=np.array([i], dtype=np.int64), **kw)
                assert r1.tobytes() == rall[i:i + 1].tobytes() and s1.tobytes() == sall[i:i + 1].tobytes(), i
    finally:
        geer.er_graph_destroy(h)


def test_dense_mode_limits(geer, tiny):
    """More than ER_DENSE_MAX_QUERIES active queries: the wave falls back to the push (same
    bits); an invalid smm_mode is rejected."""
    g, pairs = tiny
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        geer.er_graph_set_lambda(h, g.lam)
        many = np.ascontiguousarray(np.tile(pairs, (3, 1)))   # 300 queries
        out = _modes(geer, h, many, 0.05, force_ell_b=3)
        r1, s1, _, _ = out[geer.SMM_FRONTIER]
        r2, s2, d2, w2 = out[geer.SMM_DENSE]
        assert r2.tobytes() == r1.tobytes() and s2.tobytes() == s1.tobytes()
        assert d2 < w2
        with pytest.raises(geer.GeerError) as e:
            geer.er_query_batch_ex(h, pairs, 0.1, smm_mode=3)
        assert e.value.code == geer.ER_EINVAL
    finally:
        geer.er_graph_destroy(h)
