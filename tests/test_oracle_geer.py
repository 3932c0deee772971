"""Pins for the GEER / AMC / SMM oracle (oracle/geer_oracle.c).

Pinned against: Philox known-answer vectors (tests/golden/philox_kat.txt), the
paper's Fig. 3 #path rows (tests/golden/fig3_paths.txt), SPEC's hand-evaluated
closed forms, dense matrix powers of P, the K_n series
closed form, Thm 3.1's tail bound, Lemma 3.3's walk-sum interval, Eq. 12's
unbiasedness and the epsilon contract of Def. 2.2 against the exact oracle.
"""
import math
from pathlib import Path

import numpy as np
import pytest

import oracle
import workloads as W
from oracle import exact

GOLD = Path(__file__).parent / "golden"


def _rows(name):
    out = {}
    for line in (GOLD / name).read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            k, *v = line.split()
            out[k] = v
    return out


# ------------------------------------------------------------------ RNG
def test_philox_known_answers():
    for line in (GOLD / "philox_kat.txt").read_text().splitlines():
        if not line.strip() or line.startswith("#"):
            continue
        w = [int(x, 16) for x in line.split()]
        assert oracle.philox4x32_10(w[0:4], w[4:6]).tolist() == w[6:10]


# ------------------------------------------------------------------ closed forms
def test_spec_hand_values():
    # S:241-243 refined ell (Eq.6)
    assert oracle.refined_ell(2, 2, 0.1, 0.5) == 5
    assert oracle.refined_ell(2, 7, 0.5, 0.5) == 2
    # clamp at 0 when the log argument is <= 1 (R3)
    assert oracle.refined_ell(1000, 1000, 0.9, 0.5) == 0
    # S:249-251 Peng's ell (Eq.5)
    assert oracle.peng_ell(0.1, 0.5) == 6
    assert oracle.peng_ell(0.5, 0.5) == 3
    # S:257-259 psi (Eq.10)
    assert abs(oracle.psi(1, 1.0, 0.0, 1.0, 0.0, 2, 7) - 9 / 7) < 1e-15
    assert oracle.psi(0, 1.0, 0.5, 1.0, 0.5, 2, 7) == 0.0
    assert abs(oracle.psi(3, 0.2, 0.1, 0.2, 0.1, 2, 2) - 1.0) < 1e-15
    # S:265-267 eta* (Eq.9): ceil(60.90) = 61, and ln(2 tau/delta) = 1 case
    assert math.ceil(oracle.eta_star(9 / 7, 0.5, 0.1, 5)) == 61
    assert abs(oracle.eta_star(1.0, 1.0, 2 / math.e, 1) - 2.0) < 1e-12
    # S:273-275 Bernstein half-width (Eq.8)
    assert abs(oracle.bernstein_f(100, 0.04, 1.0, 0.03) - 0.198852) < 1e-6
    assert abs(oracle.bernstein_f(300, 0.0, 1.0, 0.3) - 3 * math.log(10) / 300) < 1e-15
    f100 = oracle.bernstein_f(100, 0.04, 1.0, 0.03)
    f400 = oracle.bernstein_f(400, 0.04, 1.0, 0.03)
    t1 = math.sqrt(0.08 * math.log(100) / 100)
    assert abs(f400 - (t1 / 2 + (f100 - t1) / 4)) < 1e-15
    # S:285-287 budget: eta*=61, tau=5 -> eta0=4, h=124; eta*=0 -> eta0=1; tau=1 -> eta0=eta*
    assert oracle.eta0(61.0, 5) == 4 and oracle.h_budget(4, 5) == 124
    assert oracle.eta0(0.0, 5) == 1 and oracle.h_budget(1, 5) == 31
    assert oracle.eta0(37.0, 1) == 37


def test_fig3_eta_row_alternative_form():
    # the printed eta* row follows an older psi / ln(1/delta) convention.
    row = [int(x) for x in _rows("fig3_paths.txt")["eta_row"]]
    ds, dt = 2, 7
    alt = [math.ceil(2 * (2 * lf * (1 / ds + 1 / dt)) ** 2 * math.log(1 / 0.1) / 0.5 ** 2)
           for lf in range(1, 9)]
    assert alt == row
    # ... whereas Eq.9/10 (normative) give a different row
    eq = [math.ceil(oracle.eta_star(oracle.psi(lf, 1, 0, 1, 0, ds, dt), 0.5, 0.1, 5)) for lf in range(1, 9)]
    assert eq[0] == 61 and eq != row


# ------------------------------------------------------------------ propagation / SMM
def test_fig3_path_counts():
    gold = _rows("fig3_paths.txt")
    g, idx = W.toy_fig3()
    assert oracle.walk_counts(g, idx["s"], 8) == [int(x) for x in gold["path_s"]]
    assert oracle.walk_counts(g, idx["t"], 8) == [int(x) for x in gold["path_t"]]


def test_k3_smm_spec_values():
    k3 = W.complete(3)
    assert oracle.smm(k3, 0, 1, 2)[0] == 0.75
    assert oracle.smm(k3, 0, 1, 5)[0] == 0.65625
    assert oracle.smm(k3, 1, 1, 4)[0] == 0.0           # s = t


@pytest.mark.parametrize("n", [3, 5, 10])
def test_complete_graph_series_closed_form(n):
    g = W.complete(n)
    for ell in range(0, 8):
        want = (2 / n) * (1 - (-1 / (n - 1)) ** (ell + 1))
        assert abs(oracle.smm(g, 0, 1, ell)[0] - want) < 1e-14


def test_propagation_matches_dense_matrix_powers():
    # iterated apply of P to e_u equals column/row of P^i (dense numpy), 1e-10.
    for seed in range(5):
        g = W.random_small(seed, 18, 0.2)
        P = exact.dense_P(g)
        for u in (0, 7):
            x = np.zeros(g.n)
            x[u] = 1.0
            for i in range(1, 11):
                x = oracle.propagate_dense(g, x)
                want = np.linalg.matrix_power(P, i)[:, u]   # s*(v) = p_i(v, u)
                assert np.allclose(x, want, atol=1e-12)


def test_smm_terms_match_dense_series():
    for seed in range(4):
        g = W.random_small(seed + 20, 25, 0.15)
        for s, t in [(0, 5), (3, 24), (10, 11)]:
            for ell in (0, 1, 4, 9):
                assert abs(oracle.smm(g, s, t, ell)[0] - exact.r_ell(g, s, t, ell)) < 1e-12


def test_geer_head_terms_equal_plain_smm():
    # The sparse pull inside GEER (geer_oracle.c smm_step) reproduces the dense
    # definition bit for bit (force ell_b to compare every iteration).
    g, pairs = W.tiny_er(), None
    lam = exact.lambda_dense(g)
    pairs = W.query_pairs(g, 20, 5)
    _, st = oracle.geer_batch(g, lam, pairs, 0.02, force_ell_b=6)
    for (s, t), row in zip(pairs, st):
        if s == t or row["ell_b"] == 0:
            continue
        rb, terms, _, _ = oracle.smm(g, int(s), int(t), int(row["ell_b"]))
        k = min(8, int(row["ell_b"]))
        assert np.array_equal(row["rb_terms"][:k], terms[:k])
        assert row["r_b"] == rb


def test_truncation_bound_thm31():
    # Thm 3.1 with exact lambda: |r - r_ell| <= lambda^(ell+1)/(1-lambda)(1/ds+1/dt) <= eps/2.
    for seed in range(12):
        g = W.random_small(100 + seed, 25, 0.12)
        lam = exact.lambda_dense(g)
        d = g.degrees()
        pairs = [(0, 1), (2, 17), (5, 24), (9, 13)]
        R = exact.er_pinv(g, pairs)
        for (s, t), r in zip(pairs, R):
            for eps in (0.5, 0.1):
                ell = oracle.refined_ell(d[s], d[t], eps, lam)
                rl = oracle.smm(g, s, t, ell)[0]
                tail = lam ** (ell + 1) / (1 - lam) * (1 / d[s] + 1 / d[t])
                assert abs(r - rl) <= tail + 1e-12
                assert abs(r - rl) <= eps / 2


# ------------------------------------------------------------------ walks
def test_walks_are_valid_and_uniform():
    g = W.random_small(3, 40, 0.1)
    for k in range(50):
        end, trace, _ = oracle.walk(g, 0, 25, q=7, k=k)
        prev = 0
        for v in trace:
            assert v in set(g.neighbors(prev).tolist())
            prev = int(v)
        assert end == trace[-1]
    # one-step distribution from a degree-5 node: chi-square, 10^5 draws
    g = W.star_triangle(5)
    counts = np.zeros(g.n)
    for k in range(20000):
        for side in (0, 1):
            for q in (0, 1):
                for b in (0,):
                    counts[oracle.walk(g, 0, 1, q=q, b=b, side=side, k=k)[0]] += 1
    obs = counts[1:6]
    exp = obs.sum() / 5
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert chi2 < 18.47  # df=4, p=0.001


def test_lemma33_walk_sum_and_zk_bound():
    rng = np.random.default_rng(0)
    g = W.random_small(8, 30, 0.12)
    for trial in range(30):
        x = rng.random(g.n) * (rng.random(g.n) < 0.5)
        lf = int(rng.integers(1, 12))
        srt = np.sort(x)[::-1]
        lo = lf * x.min()
        hi = math.ceil(lf / 2) * srt[0] + math.floor(lf / 2) * srt[1]
        for k in range(60):
            _, trace, acc = oracle.walk(g, int(rng.integers(0, g.n)), lf, k=k, q=trial, y=x)
            assert lo - 1e-12 <= acc <= hi + 1e-12
            assert abs(acc - x[trace].sum()) < 1e-12
    # |Z_k| <= psi/2 for the GEER hand-off vectors
    g = W.tiny_er()
    s, t = 4, 777
    for lb in (1, 2):
        _, _, xs, xt = oracle.smm(g, s, t, lb)
        d = g.degrees()
        for lf in (1, 2, 5):
            m = lambda v: np.sort(v)[::-1][:2]
            (a1, a2), (b1, b2) = m(xs), m(xt)
            psi = oracle.psi(lf, a1, a2, b1, b2, d[s], d[t])
            z = oracle.amc_samples(g, s, t, xs, xt, lf, 20000)
            assert np.abs(z).max() <= psi / 2 + 1e-12


@pytest.mark.parametrize("case", ["k3", "rand"])
def test_unbiasedness_eq12(case):
    if case == "k3":
        g, s, t = W.complete(3), 0, 1
        xs = np.eye(3)[0]
        xt = np.eye(3)[1]
        lf = 3
    else:
        g, s, t = W.random_small(4, 20, 0.2), 2, 15
        _, _, xs, xt = oracle.smm(g, s, t, 1)
        lf = 4
    z = oracle.amc_samples(g, s, t, xs, xt, lf, 100000, q=3)
    q = exact.q_st(g, s, t, xs, xt, lf)
    se = z.std() / math.sqrt(len(z))
    assert abs(z.mean() - q) <= 4 * se + 1e-15


def test_geer_decomposition_exact():
    # r_b + q(s*, t*, ell - ell_b) = r_ell (Eq.14 with P:554-560's rewrite of r*_f).
    g = W.random_small(9, 25, 0.15)
    for s, t in [(0, 3), (7, 20)]:
        for ell, lb in [(6, 1), (6, 3), (9, 2)]:
            rb, _, xs, xt = oracle.smm(g, s, t, lb)
            assert abs(rb + exact.q_st(g, s, t, xs, xt, ell - lb) - exact.r_ell(g, s, t, ell)) < 1e-12


# ------------------------------------------------------------------ GEER end to end
def test_geer_tiny_within_eps_of_exact(tiny):
    g, pairs = tiny
    ex = exact.er_pinv(g, pairs)
    for eps in (0.1, 0.5):
        r, st = oracle.geer_batch(g, g.lam, pairs, eps)
        assert np.abs(r - ex).max() <= eps
        # budget accounting: walks = eta0 (2^b - 1) <= h, steps = 2 walks lf
        amc = st["ell_f"] > 0
        b = st["batches_run"][amc]
        assert np.array_equal(st["walks_total"][amc], st["eta0"][amc] * (2 ** b - 1))
        assert np.array_equal(st["steps_total"], 2 * st["walks_total"] * st["ell_f"])
        assert (st["ell_b"][amc] >= 1).all()                     # repeat...until (R4)
        assert (st["ell_b"] <= st["ell"]).all()
        assert np.allclose(r, st["r_b"] + st["r_f"], atol=0, rtol=0)


def test_geer_amc_only_and_edge_cases():
    g = W.lollipop(5)
    lam = exact.lambda_dense(g)
    pairs = np.array([[0, 7], [3, 3], [1, 2], [7, 0]], dtype=np.int32)
    ex = exact.er_pinv(g, pairs)
    r, st = oracle.geer_batch(g, lam, pairs, 0.2)
    assert r[1] == 0.0 and st["ell"][1] == 0
    assert np.abs(r - ex).max() <= 0.2
    r0, st0 = oracle.geer_batch(g, lam, pairs, 0.2, force_ell_b=0)   # AMC alone (Thm 3.4)
    assert (st0["ell_b"] == 0).all() and np.abs(r0 - ex).max() <= 0.2
    # ell = 0 returns r_b = 1/ds + 1/dt exactly (R3)
    k = W.complete(30)
    r, st = oracle.geer_batch(k, 1 / 29, [[0, 1]], 0.9)
    assert st["ell"][0] == 0 and r[0] == 1 / 29 + 1 / 29
    with pytest.raises(ValueError):
        oracle.geer_batch(k, 1 / 29, [[0, 30]], 0.1)
    with pytest.raises(ValueError):
        oracle.geer_batch(k, 1.0, [[0, 1]], 0.1)


@pytest.mark.parametrize("gname", ["k3", "lollipop", "rand100"])
def test_eps_success_frequency(gname):
    # Thm 3.4 / Def. 2.2: |r' - r| <= eps with prob >= 1 - delta; 200 seeded runs, delta=0.1.
    g = {"k3": W.complete(3), "lollipop": W.lollipop(4), "rand100": W.random_small(42, 100, 0.04)}[gname]
    lam = exact.lambda_dense(g)
    pair = (0, 1) if gname == "k3" else (0, g.n - 1)
    ex = exact.er_pinv(g, [pair])[0]
    pairs = np.tile(np.array(pair, dtype=np.int32), (200, 1))
    for eps in (0.5, 0.2):
        r, _ = oracle.geer_batch(g, lam, pairs, eps, delta=0.1, seed=99)
        assert (np.abs(r - ex) <= eps).mean() >= 0.9


def test_deterministic_across_threads(tiny):
    g, pairs = tiny
    a, sa = oracle.geer_batch(g, g.lam, pairs, 0.1, nthreads=1)
    b, sb = oracle.geer_batch(g, g.lam, pairs, 0.1, nthreads=4)
    assert a.tobytes() == b.tobytes() and sa.tobytes() == sb.tobytes()
    # query_index_base shifts the RNG stream (different walks), not the head
    c, sc = oracle.geer_batch(g, g.lam, pairs, 0.1, query_index_base=1000)
    assert np.array_equal(sa["ell_b"], sc["ell_b"]) and not np.array_equal(a, c)


def test_walk_checksum_is_sum_of_endpoint_hashes():
    g = W.lollipop(5)
    lam = exact.lambda_dense(g)
    _, st = oracle.geer_batch(g, lam, [[0, 7]], 0.3, query_index_base=5)
    row = st[0]
    lf = int(row["ell_f"])
    assert lf > 0
    # rebuild y from the head vectors, then recount every walk's endpoint
    _, _, xs, xt = oracle.smm(g, 0, 7, int(row["ell_b"]))
    ck = 0
    for b in range(int(row["batches_run"])):
        for k in range(int(row["eta0"]) << b):
            e0 = oracle.walk(g, 0, lf, q=5, b=b, side=0, k=k)[0]
            e1 = oracle.walk(g, 7, lf, q=5, b=b, side=1, k=k)[0]
            ck = (ck + oracle.walk_hash(5, b, 0, k, e0) + oracle.walk_hash(5, b, 1, k, e1)) % 2 ** 64
    assert ck == int(row["walk_checksum"])


def test_variant_switch_ratio_extremes(tiny):
    """SURVEY 8(f)#4 GPU-cost switch knob: ratio -> infinity never leaves the SMM head (ell_b = ell,
    r' = r_ell by dense matrix powers, Eq. 4); ratio 0 leaves after the first iteration; 1.0 is
    Eq. 15 (the default)."""
    g, pairs = tiny
    sub = pairs[:12]
    r_inf, st_inf = oracle.geer_batch(g, g.lam, sub, 0.1, switch_ratio=1e18)
    assert np.array_equal(st_inf["ell_b"], st_inf["ell"]) and (st_inf["batches_run"] == 0).all()
    for (s, t), r, L in zip(sub, r_inf, st_inf["ell"]):
        assert abs(r - exact.r_ell(g, int(s), int(t), int(L))) <= 1e-12
    _, st0 = oracle.geer_batch(g, g.lam, sub, 0.1, switch_ratio=0.0)
    assert ((st0["ell_b"] == 1) | (st0["ell"] == 0)).all()
    r1, st1 = oracle.geer_batch(g, g.lam, sub, 0.1, switch_ratio=1.0)
    rd, sd = oracle.geer_batch(g, g.lam, sub, 0.1)
    assert r1.tobytes() == rd.tobytes()


def test_variant_reuse_samples_is_running_mean(tiny):
    """SURVEY 8(f)#4 sample-reuse knob: the final estimate is r_b + the mean of Z_0..Z_{eta-1} of
    ONE sample stream (batch key 0), eta = the last batch size; walks are never redrawn."""
    g, pairs = tiny
    sub = pairs[:30]
    r, st = oracle.geer_batch(g, g.lam, sub, 0.1, reuse_samples=1)
    checked = 0
    for i, ((s, t), ri) in enumerate(zip(sub, r)):
        lf = int(st["ell_f"][i])
        if lf <= 0:
            continue
        eta_last = int(st["eta0"][i]) << (int(st["batches_run"][i]) - 1)
        assert int(st["walks_total"][i]) == eta_last
        rb, _, xs, xt = oracle.smm(g, int(s), int(t), int(st["ell_b"][i]))
        z = oracle.amc_samples(g, int(s), int(t), xs, xt, lf, eta_last, q=i, b=0)
        acc = 0.0
        for zk in z:
            acc += zk
        assert ri == rb + acc / eta_last
        checked += 1
    assert checked > 10
