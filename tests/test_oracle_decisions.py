"""Pins for the oracle's GEER decisions that are not closed-form helpers: the top-2 statistics
and psi fed to Eq. 9 inside the SMM loop, Eq. 15's switch (strict inequality, current iterate),
and the Bernstein stop of Alg. 1 L13 with f(eta, sigma^2, psi, delta/tau) <= eps/2.

Each expected value comes from something other than the oracle's own loop:
  * hand-evaluated SMM iterates of K_n and of a star with a triangle (closed forms written out
    below), which fix max_1 = max_2 ties, a one-hot second maximum of 0, vol and the r_b terms;
  * an exact vol == h construction on K_32, which separates Eq. 15's `vol > h` from `>=`;
  * the plain dense SMM (oracle.smm, matrix-free P applied to the whole vector) at every
    iteration, from which vol, top-2, psi, eta0, h and the first iteration with vol > h are
    rebuilt with numpy;
  * the walk samples of every batch (oracle.amc_samples, same Philox keys), from which Z,
    sigma^2, f with delta/tau and the stopping batch are rebuilt.
P:n = PAPER.md line n: max_k, Eq. 10, Eq. 9, Eq. 15,
Alg. 3 L9, Alg. 1 L11-L14, Eq. 8.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W

TAU, DELTA = 5, 0.01


def eq10_psi(lf, m1s, m2s, m1t, m2t, ds, dt):
    # Eq. 10, written out: 2 ceil(lf/2) (m1s/ds + m1t/dt) + 2 floor(lf/2) (m2s/ds + m2t/dt)
    return 2.0 * float((lf + 1) // 2) * (m1s / ds + m1t / dt) + 2.0 * float(lf // 2) * (m2s / ds + m2t / dt)


def eta0_h(psi, eps, delta=DELTA, tau=TAU):
    # Eq. 9 eta* = 2 psi^2 ln(2 tau / delta) / eps^2; eta0 = max(1, ceil(eta* / 2^(tau-1)))
    # (R6); h = (2^tau - 1) eta0
    es = 2.0 * psi * psi * math.log(2.0 * tau / delta) / (eps * eps)
    e0 = max(1, math.ceil(es / 2 ** (tau - 1)))
    return e0, (2 ** tau - 1) * e0


def run(g, lam, pairs, eps, **kw):
    return oracle.geer_batch(g, lam, np.asarray(pairs, dtype=np.int32), eps, delta=DELTA, tau=TAU, **kw)


# ------------------------------------------------------------------ hand-evaluated iterates
@pytest.mark.parametrize("n", [6, 11, 32])
def test_complete_graph_iterates_ties_and_vol(n):
    """K_n, s = 0, t = 1.  Iteration 1: s* = 1/(n-1) on V \\ {s} (n-1 equal entries, so
    max_2 = max_1 = 1/(n-1), R5); vol = 2 (n-1)^2.  Iteration 2: s*(s) = 1/(n-1), every other
    entry (n-2)/(n-1)^2; vol = 2 n (n-1).  t* mirrors s*."""
    g = W.complete(n)
    lam = 0.8   # an upper bound on K_n's 1/(n-1) (any lambda' >= lambda keeps Thm 3.1, R12): longer ell
    eps = 0.01
    d = n - 1
    for lb, (m1, m2, vol) in {1: (1 / d, 1 / d, 2 * d * d), 2: (1 / d, (n - 2) / d ** 2, 2 * n * d)}.items():
        _, st = run(g, lam, [[0, 1]], eps, force_ell_b=lb)
        row = st[0]
        ell = int(row["ell"])
        assert ell >= lb + 2, "need lf >= 2 so that max_2 enters psi"
        assert row["ell_b"] == lb and row["vol_last"] == vol
        psi = eq10_psi(ell - lb, m1, m2, m1, m2, d, d)
        assert row["psi"] == pytest.approx(psi, rel=1e-14, abs=0)
        # a top-2 that took the second DISTINCT value would see max_2 = 0 at iteration 1
        wrong = eq10_psi(ell - lb, m1, 0.0, m1, 0.0, d, d)
        assert abs(row["psi"] - wrong) > 1e-3 * psi
        e0, h = eta0_h(psi, eps)
        assert row["eta0"] == e0 and row["h_last"] == h


def test_star_triangle_iterates_one_hot_and_terms():
    """Star with centre 0 and leaves 1..L plus the edge (1,2); s = 0 (d = L), t = 3 (d = 1).
    Iteration 1: s* = 1/2 on {1, 2}, 1 on the other leaves (max_1 = max_2 = 1); t* = (1/L) e_0
    (one nonzero entry: max_2 = 0); vol = (L-2) + 4 + L; r_b term = -1/L - 1/L.
    Iteration 2: s* = (L-1)/L at 0, 1/4 at 1 and 2; t* = 1/(2L) at 1, 2 and 1/L at the other
    leaves; vol = (L + 4) + (L + 2)."""
    L = 9
    g = W.star_triangle(L)
    lam = 0.9
    eps = 0.02
    ds, dt = float(L), 1.0
    it = {1: (1.0, 1.0, 1 / L, 0.0, (L - 2) + 4 + L),
          2: ((L - 1) / L, 0.25, 1 / L, 1 / L, (L + 4) + (L + 2))}
    for lb, (m1s, m2s, m1t, m2t, vol) in it.items():
        _, st = run(g, lam, [[0, 3]], eps, force_ell_b=lb)
        row = st[0]
        ell = int(row["ell"])
        assert ell > lb and row["ell_b"] == lb and row["vol_last"] == vol
        psi = eq10_psi(ell - lb, m1s, m2s, m1t, m2t, ds, dt)
        assert row["psi"] == pytest.approx(psi, rel=1e-14, abs=0)
        e0, h = eta0_h(psi, eps)
        assert row["eta0"] == e0 and row["h_last"] == h
    # series terms: iteration 1 = s*(s)/ds + t*(t)/dt - s*(t)/ds - t*(s)/dt = 0 + 0 - 1/L - 1/L;
    # iteration 2 = s*_2(0)/L + t*_2(3)/1 - s*_2(3)/L - t*_2(0)/1 = ((L-1)/L)/L + 1/L - 0 - 0
    _, st = run(g, lam, [[0, 3]], eps, force_ell_b=2)
    assert st[0]["rb_terms"][0] == pytest.approx(-2.0 / L, rel=1e-15)
    assert st[0]["rb_terms"][1] == pytest.approx(((L - 1) / L) / L + 1.0 / L, rel=1e-15)


# ------------------------------------------------------------------ Eq. 15 at equality
def _k32_lambda_for_ell(eps, want_ell):
    """A lambda in (0,1) for which Eq. 6 gives ell = want_ell on K_32 (d = 31) at this eps."""
    for lam in np.linspace(0.02, 0.98, 4801):
        if oracle.refined_ell(31, 31, eps, float(lam)) == want_ell:
            return float(lam)
    raise AssertionError("no lambda found")


@pytest.mark.parametrize("eta_star,want_eta0,want_ell_b", [(984.0, 62, 2), (970.0, 61, 1)])
def test_eq15_strict_inequality_at_equality(eta_star, want_eta0, want_ell_b):
    """K_32, s = 0, t = 1, ell = 3.  After iteration 1 vol = 2 * 31^2 = 1922 = 31 * 62 (above).
    eps is chosen so that eta* = eta_star at lf = 2 (psi = 8/961): eta* = 984 gives eta0 = 62 and
    h = 1922 = vol, so Eq. 15's `vol > h` is false and the head continues (ell_b = 2; a `>=`
    would stop at 1); eta* = 970 gives eta0 = 61, h = 1891 < vol, so it stops at ell_b = 1."""
    g = W.complete(32)
    psi1 = 8.0 / 961.0
    eps = math.sqrt(2.0 * psi1 * psi1 * math.log(2.0 * TAU / DELTA) / eta_star)
    lam = _k32_lambda_for_ell(eps, 3)
    _, st1 = run(g, lam, [[0, 1]], eps, force_ell_b=1)
    assert st1[0]["ell"] == 3 and st1[0]["vol_last"] == 1922
    assert st1[0]["eta0"] == want_eta0 and st1[0]["h_last"] == 31 * want_eta0
    _, st = run(g, lam, [[0, 1]], eps)
    assert st[0]["ell_b"] == want_ell_b


# ------------------------------------------------------------------ rebuilt from the plain SMM
def _rebuild_head(g, s, t, ell, eps, max_it=None):
    """Alg. 3 L5-L9 rebuilt from oracle.smm's dense vectors: (ell_b, vol, h, psi, eta0)."""
    d = g.degrees()
    ds, dt = float(d[s]), float(d[t])
    lb = 0
    while True:
        lb += 1
        _, _, xs, xt = oracle.smm(g, s, t, lb)
        vol = int(d[xs != 0.0].sum() + d[xt != 0.0].sum())
        srt_s = np.sort(xs)[::-1]
        srt_t = np.sort(xt)[::-1]
        psi = eq10_psi(ell - lb, srt_s[0], srt_s[1], srt_t[0], srt_t[1], ds, dt)
        e0, h = eta0_h(psi, eps)
        if vol > h or lb >= ell:
            return lb, vol, h, psi, e0


@pytest.mark.parametrize("eps", [0.1, 0.05])
def test_head_decisions_rebuilt_from_dense_smm(eps):
    g = W.rmat(12, 5, seed=77)
    lam = W.lambda_of(g)
    pairs = W.query_pairs(g, 60, seed=78)
    _, st = run(g, lam, pairs, eps)
    checked = 0
    for (s, t), row in zip(pairs, st):
        s, t = int(s), int(t)
        if s == t or row["ell"] == 0:
            continue
        lb, vol, h, psi, e0 = _rebuild_head(g, s, t, int(row["ell"]), eps)
        assert row["ell_b"] == lb and row["vol_last"] == vol and row["h_last"] == h
        if row["ell_f"] > 0:
            assert row["psi"] == psi and row["eta0"] == e0
        checked += 1
    assert checked >= 50


# ------------------------------------------------------------------ Bernstein stop, rebuilt
def _rebuild_amc(g, s, t, q, lb, lf, psi, eta0, eps):
    """Alg. 1 L4-L14 rebuilt from the batch samples: fresh samples per batch (R8), Z and the
    one-pass sigma^2 (R7), f = Eq. 8 with d = delta/tau (Alg. 1 L13), stop at f <= eps/2."""
    _, _, xs, xt = oracle.smm(g, s, t, lb)
    Lb = math.log(3.0 / (DELTA / TAU))
    walks = 0
    for b in range(TAU):
        eta = eta0 << b
        z = oracle.amc_samples(g, s, t, xs, xt, lf, eta, q=q, b=b)
        s1 = s2 = 0.0
        for zk in z:   # sequential, sample order
            s1 += zk
            s2 += zk * zk
        Z = s1 / eta
        var = max(0.0, s2 / eta - Z * Z)
        f = math.sqrt(2.0 * var * Lb / eta) + 3.0 * psi * Lb / eta
        walks += eta
        if f <= eps / 2.0 or b == TAU - 1:
            return b + 1, f, Z, var, walks


@pytest.mark.parametrize("eps", [0.1, 0.3])
def test_bernstein_stop_rebuilt_from_samples(tiny, eps):
    g, pairs = tiny
    _, st = run(g, g.lam, pairs[:40], eps, query_index_base=500)
    checked = 0
    for i, ((s, t), row) in enumerate(zip(pairs[:40], st)):
        lf = int(row["ell_f"])
        if s == t or lf <= 0:
            continue
        br, f, Z, var, walks = _rebuild_amc(g, int(s), int(t), 500 + i, int(row["ell_b"]), lf, float(row["psi"]),
                                            int(row["eta0"]), eps)
        assert row["batches_run"] == br and row["walks_total"] == walks
        assert row["f_last"] == f and row["r_f"] == Z and row["sigma2_last"] == var
        checked += 1
    assert checked >= 20
    # the stop uses delta/tau: with delta in place of delta/tau some query would stop earlier
    Lwrong = math.log(3.0 / DELTA)
    assert Lwrong < math.log(3.0 / (DELTA / TAU))
