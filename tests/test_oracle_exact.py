"""Pins for the exact-ER oracle (oracle/exact.py) and lambda.

Every check is against something other than the oracle itself: closed forms of
resistor networks, Foster's theorem, the grounded-Laplacian route, and known
spectra.  PAPER.md citations: Def. 2.1 / Eq. 1, r = c/(2m),
1/(2m) <= r <= 1 on edges, lambda = max(|lambda_2|, |lambda_n|).
"""
import itertools
import math

import numpy as np
import pytest

import workloads as W
from oracle import exact


@pytest.mark.parametrize("n", [3, 5, 10])
def test_complete_graph_2_over_n(n):
    g = W.complete(n)
    pairs = [(i, j) for i in range(n) for j in range(n) if i != j]
    assert np.allclose(exact.er_pinv(g, pairs), 2.0 / n, atol=1e-12)
    assert np.allclose(exact.er_grounded(g, pairs), 2.0 / n, atol=1e-12)


@pytest.mark.parametrize("n", [5, 9, 15])
def test_odd_cycle(n):
    g = W.cycle(n)
    pairs = [(0, k) for k in range(n)]
    want = [k * (n - k) / n for k in range(n)]
    assert np.allclose(exact.er_pinv(g, pairs), want, atol=1e-11)


def test_path_is_hop_distance_and_triangle_two_thirds():
    g = W.path(7)
    pairs = [(i, j) for i in range(7) for j in range(7)]
    assert np.allclose(exact.er_pinv(g, pairs), [abs(i - j) for i, j in pairs], atol=1e-10)
    # K3 adjacent pair 2/3, path u-v-w r(u,w) = 2.
    assert abs(exact.er_pinv(W.complete(3), [(0, 1)])[0] - 2 / 3) < 1e-12
    assert abs(exact.er_pinv(W.path(3), [(0, 2)])[0] - 2.0) < 1e-12


def test_tree_is_path_length():
    rng = np.random.default_rng(7)
    n = 40
    parent = [int(rng.integers(0, i)) for i in range(1, n)]
    g = W.from_edges(n, [(i + 1, p) for i, p in enumerate(parent)])
    # hop distance by BFS
    def bfs(s):
        d = -np.ones(n, dtype=int)
        d[s] = 0
        q = [s]
        while q:
            v = q.pop(0)
            for w in g.neighbors(v):
                if d[w] < 0:
                    d[w] = d[v] + 1
                    q.append(int(w))
        return d
    D = np.array([bfs(s) for s in range(n)])
    pairs = list(itertools.product(range(0, n, 3), range(n)))
    got = exact.er_pinv(g, pairs)
    assert np.allclose(got, [D[s, t] for s, t in pairs], atol=1e-9)


def test_lollipop_cactus_sum():
    # ER on a cactus = sum of block ERs: across the triangle 2/3, along the path 1 per hop.
    g = W.lollipop(6)
    tail = 3 + 5  # last path node
    assert abs(exact.er_pinv(g, [(0, tail)])[0] - (2 / 3 + 6)) < 1e-10
    assert abs(exact.er_pinv(g, [(2, tail)])[0] - 6.0) < 1e-10


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_foster_symmetry_triangle_edge_bounds(seed):
    g = W.random_small(seed, 30, 0.15)
    n = g.n
    edges = [(u, int(v)) for u in range(n) for v in g.neighbors(u) if u < v]
    R = exact.er_pinv(g, [(s, t) for s in range(n) for t in range(n)]).reshape(n, n)
    # Foster's theorem: sum over edges of r(u,v) = n - 1.
    assert abs(sum(R[u, v] for u, v in edges) - (n - 1)) < 1e-9
    assert np.allclose(R, R.T, atol=1e-12)
    assert np.allclose(np.diag(R), 0.0, atol=1e-12)
    # triangle inequality (ER is a metric)
    assert (R[:, :, None] <= R[:, None, :] + R.T[None, :, :] + 1e-10).all()
    # 1/(2m) <= r(s,t) <= 1 for (s,t) in E
    m = len(edges)
    er = np.array([R[u, v] for u, v in edges])
    assert (er >= 1 / (2 * m) - 1e-12).all() and (er <= 1 + 1e-12).all()
    # pinv and grounded solves agree
    pairs = [(0, 5), (3, 17), (29, 1)]
    assert np.allclose(exact.er_pinv(g, pairs), exact.er_grounded(g, pairs, ground=11), atol=1e-10)


def test_commute_time_identity_small():
    # r(s,t) = c(s,t)/(2m): c from hitting times by linear solves.
    g = W.random_small(5, 12, 0.3)
    n = g.n
    P = exact.dense_P(g)
    m = g.m

    def hitting(target):
        idx = [i for i in range(n) if i != target]
        M = np.eye(n - 1) - P[np.ix_(idx, idx)]
        h = np.linalg.solve(M, np.ones(n - 1))
        out = np.zeros(n)
        out[idx] = h
        return out
    for s, t in [(0, 7), (3, 11)]:
        c = hitting(t)[s] + hitting(s)[t]
        assert abs(c / (2 * m) - exact.er_pinv(g, [(s, t)])[0]) < 1e-9


@pytest.mark.parametrize("n", [3, 4, 6])
def test_lambda_complete(n):
    assert abs(exact.lambda_dense(W.complete(n)) - 1.0 / (n - 1)) < 1e-12


@pytest.mark.parametrize("n", [5, 7, 11])
def test_lambda_odd_cycle(n):
    assert abs(exact.lambda_dense(W.cycle(n)) - math.cos(math.pi / n)) < 1e-12


def test_lambda_petersen_and_arpack_matches_dense(tiny):
    assert abs(exact.lambda_dense(W.petersen()) - 2.0 / 3.0) < 1e-12
    g, _ = tiny
    assert abs(W.lambda_of(g) - exact.lambda_dense(g)) < 1e-8
    assert abs(g.lam - exact.lambda_dense(g)) < 1e-8


def test_spectral_identity_eq17():
    # Lemma A.1 Eq.17: 1/pi(v) = sum_k f_k(v)^2 with f_k pi-orthonormal.
    g = W.random_small(11, 20, 0.25)
    d = exact.degrees(g)
    A = exact.dense_A(g)
    N = A / np.sqrt(d)[:, None] / np.sqrt(d)[None, :]
    w, V = np.linalg.eigh(N)
    pi = d / d.sum()
    F = V / np.sqrt(pi)[:, None]          # f_k = D^-1/2 w_k rescaled to pi-orthonormal
    assert np.allclose((F ** 2).sum(1), 1.0 / pi, atol=1e-8)
    # Eq.16: p_i(u,v) = sum_k f_k(u) f_k(v) pi(v) lambda_k^i
    P = exact.dense_P(g)
    for i in (1, 2, 3, 5):
        Pi = np.linalg.matrix_power(P, i)
        recon = (F * w ** i) @ F.T * pi[None, :]
        assert np.allclose(Pi, recon, atol=1e-8)


def test_series_signed_matches_matrix_powers_and_converges():
    """oracle.series_signed (sparse pull, signed vector) equals Eq. 4 by dense matrix powers
    (exact.r_ell) and converges to the exact ER (Thm 3.1) on small non-bipartite graphs."""
    import oracle
    import workloads as W
    for g, pairs in ((W.random_small(2, 40, 0.12), [(0, 5), (3, 17), (9, 9)]), (W.lollipop(6), [(0, 8), (1, 4)]),
                     (W.petersen(), [(0, 7)])):
        for s, t in pairs:
            for L in (0, 1, 4, 9):
                assert abs(oracle.series_signed(g, s, t, L) - exact.r_ell(g, s, t, L)) <= 1e-12
            if s != t:
                # Thm 3.1: with L = Eq. 6's ell at eps = 1e-10 the tail is <= 1e-10
                lam = exact.lambda_dense(g)
                L = oracle.refined_ell(int(g.degrees()[s]), int(g.degrees()[t]), 1e-10, lam)
                r = exact.er_pinv(g, np.array([[s, t]]))[0]
                assert abs(oracle.series_signed(g, s, t, L) - r) <= 1e-10 + 1e-12 * r
