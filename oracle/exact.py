"""Exact effective resistance and dense spectral helpers (oracle part c1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``er_pinv``: Def. 2.1 / Eq. 1,
  ``r(s,t) = (e_s - e_t) L^+ (e_s - e_t)^T`` with ``L^+`` the Moore-Penrose
  pseudo-inverse of ``D - A`` (numpy ``pinv``, fp64).
* ``er_grounded``: the same quantity by a grounded-Laplacian solve (a second,
  independent route used to cross-check ``er_pinv``).
* ``dense_P`` / ``lambda_dense``: ``P = D^-1 A`` and
  ``lambda = max(|lambda_2|, |lambda_n|)`` (Eq. 6) from the symmetric
  ``N = D^-1/2 A D^-1/2`` which has the same spectrum.
* ``q_st``: Eq. 11 by dense matrix powers, the expectation of Z_k (Eq. 12).
* ``r_ell``: Eq. 4 by dense matrix powers.
"""
from __future__ import annotations

import numpy as np


def dense_A(g) -> np.ndarray:
    A = np.zeros((g.n, g.n))
    for u in range(g.n):
        A[u, g.cols[g.offsets[u]:g.offsets[u + 1]]] = 1.0
    return A


def degrees(g) -> np.ndarray:
    return np.diff(np.asarray(g.offsets)).astype(np.float64)


def dense_P(g) -> np.ndarray:
    """P = D^-1 A, row-stochastic (reading R1 of DESIGN.md)."""
    return dense_A(g) / degrees(g)[:, None]


def laplacian(g) -> np.ndarray:
    A = dense_A(g)
    return np.diag(A.sum(1)) - A


def er_pinv(g, pairs) -> np.ndarray:
    Lp = np.linalg.pinv(laplacian(g), hermitian=True)
    pairs = np.asarray(pairs).reshape(-1, 2)
    s, t = pairs[:, 0], pairs[:, 1]
    return Lp[s, s] + Lp[t, t] - Lp[s, t] - Lp[t, s]


def er_grounded(g, pairs, ground=None) -> np.ndarray:
    """r(s,t) via L_g x = e_s - e_t with one node grounded (row/col removed)."""
    L = laplacian(g)
    n = g.n
    pairs = np.asarray(pairs).reshape(-1, 2)
    ground = n - 1 if ground is None else ground
    keep = np.array([i for i in range(n) if i != ground])
    Lg = L[np.ix_(keep, keep)]
    C = np.linalg.cholesky(Lg)
    pos = -np.ones(n, dtype=np.int64)
    pos[keep] = np.arange(n - 1)
    out = np.zeros(len(pairs))
    for i, (s, t) in enumerate(pairs):
        b = np.zeros(n - 1)
        if pos[s] >= 0:
            b[pos[s]] += 1.0
        if pos[t] >= 0:
            b[pos[t]] -= 1.0
        x = np.linalg.solve(C.T, np.linalg.solve(C, b))
        xs = x[pos[s]] if pos[s] >= 0 else 0.0
        xt = x[pos[t]] if pos[t] >= 0 else 0.0
        out[i] = xs - xt
    return out


def spectrum_P(g) -> np.ndarray:
    d = degrees(g)
    A = dense_A(g)
    N = A / np.sqrt(d)[:, None] / np.sqrt(d)[None, :]
    return np.sort(np.linalg.eigvalsh(N))[::-1]


def lambda_dense(g) -> float:
    ev = spectrum_P(g)
    return float(max(abs(ev[1]), abs(ev[-1])))


def r_ell(g, s, t, ell) -> float:
    """Eq. 4: sum_{i=0..ell} p_i(s,s)/d(s) + p_i(t,t)/d(t) - p_i(s,t)/d(t) - p_i(t,s)/d(s)."""
    P = dense_P(g)
    d = degrees(g)
    Pi = np.eye(g.n)
    total = 0.0
    for _ in range(ell + 1):
        total += Pi[s, s] / d[s] + Pi[t, t] / d[t] - Pi[s, t] / d[t] - Pi[t, s] / d[s]
        Pi = Pi @ P
    return float(total)


def q_st(g, s, t, xs, xt, lf) -> float:
    """Eq. 11: sum_{i=1..lf} sum_v (p_i(s,v) - p_i(t,v)) (xs(v)/d(s) - xt(v)/d(t))."""
    P = dense_P(g)
    d = degrees(g)
    y = np.asarray(xs) / d[s] - np.asarray(xt) / d[t]
    Pi = np.eye(g.n)
    total = 0.0
    for _ in range(lf):
        Pi = Pi @ P
        total += float((Pi[s] - Pi[t]) @ y)
    return total
