"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Acceptance (BASELINE north_star), per query, same (lambda, seed,
tau, query_index_base) on both sides:
  decisions         ell, ell_b, ell_f, batches_run, eta0, vol_last, h_last equal
  walks             walks_total, steps_total, walk_checksum equal (endpoints bit-exact)
  series terms      rb_terms / r_b within 1e-10 * max(|term|, 1/d_s + 1/d_t);
                    bit-exact on sorted-adjacency graphs (strict summation order, R13)
  final estimate    |r'_gpu - r'_oracle| <= 1e-9
  tiny graph        |r'_gpu - r_exact| <= eps on every pair
Queries whose tie_flags are set on either side are excluded from the exact
decision comparison (R15); the test asserts there are none on these inputs.
"""
import numpy as np
import pytest

import oracle
import workloads as W
from oracle import exact

pytestmark = pytest.mark.gpu

DECISIONS = ["ell", "ell_b", "ell_f", "batches_run", "eta0", "vol_last", "h_last",
             "walks_total", "steps_total", "walk_checksum"]


def compare(g, pairs, r_gpu, st_gpu, r_or, st_or, sorted_adj=True):
    ties = (st_gpu["tie_flags"] | st_or["tie_flags"]) != 0
    assert ties.sum() == 0, f"{ties.sum()} decision ties"
    for f in DECISIONS:
        bad = np.nonzero(st_gpu[f] != st_or[f])[0]
        assert len(bad) == 0, f"{f} differs at {bad[:5]}: gpu {st_gpu[f][bad[:5]]} oracle {st_or[f][bad[:5]]}"
    d = g.degrees()
    scale = 1.0 / d[pairs[:, 0]] + 1.0 / d[pairs[:, 1]]
    tol = 1e-10 * np.maximum(np.abs(st_or["rb_terms"]), scale[:, None])
    assert (np.abs(st_gpu["rb_terms"] - st_or["rb_terms"]) <= tol).all()
    assert (np.abs(st_gpu["r_b"] - st_or["r_b"]) <= 1e-10 * np.maximum(np.abs(st_or["r_b"]), scale)).all()
    if sorted_adj:
        assert np.array_equal(st_gpu["r_b"], st_or["r_b"]) and np.array_equal(st_gpu["psi"], st_or["psi"])
    err = np.abs(r_gpu - r_or)
    assert err.max() <= 1e-9, f"max |r_gpu - r_oracle| = {err.max()}"
    return err.max()


def run_both(G, h, g, pairs, eps, **kw):
    r, st = G.er_query_batch_ex(h, pairs, eps, 0.01, stats=True, **kw)
    okw = {k: v for k, v in kw.items() if k in ("tau", "seed", "query_index_base", "force_ell_b", "ell_variant",
                                                "switch_ratio", "reuse_samples")}
    ro, so = oracle.geer_batch(g, g.lam, pairs, eps, delta=0.01, **okw)
    return r, st, ro, so


@pytest.fixture(scope="module")
def tiny_h(geer, tiny):
    g, pairs = tiny
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    geer.er_graph_set_lambda(h, g.lam)
    yield h
    geer.er_graph_destroy(h)


@pytest.mark.parametrize("eps", [0.5, 0.1, 0.05, 0.02, 0.01])
def test_tiny_parity_and_exact(geer, tiny, tiny_h, eps):
    g, pairs = tiny
    r, st, ro, so = run_both(geer, tiny_h, g, pairs, eps)
    compare(g, pairs, r, st, ro, so)
    ex = exact.er_pinv(g, pairs)
    assert np.abs(r - ex).max() <= eps
    assert (st["steps_total"] > 0).any()


@pytest.mark.parametrize("kw", [dict(tau=1), dict(tau=8), dict(force_ell_b=0), dict(force_ell_b=3),
                                dict(ell_variant=1), dict(seed=12345, query_index_base=777),
                                dict(switch_ratio=0.25), dict(switch_ratio=4.0), dict(reuse_samples=1),
                                dict(reuse_samples=1, force_ell_b=0, tau=7)])
def test_tiny_parity_options(geer, tiny, tiny_h, kw):
    g, pairs = tiny
    r, st, ro, so = run_both(geer, tiny_h, g, pairs, 0.2, **kw)
    compare(g, pairs, r, st, ro, so)


def test_tiny_determinism_sharding_device_pointers(geer, tiny, tiny_h):
    import torch
    g, pairs = tiny
    a, _ = geer.er_query_batch_ex(tiny_h, pairs, 0.1)
    b, _ = geer.er_query_batch_ex(tiny_h, pairs, 0.1)
    assert a.tobytes() == b.tobytes()
    # sharding by query_index_base reproduces the unsharded batch bit for bit
    parts = [geer.er_query_batch_ex(tiny_h, pairs[lo:hi], 0.1, query_index_base=lo)[0]
             for lo, hi in [(0, 37), (37, 64), (64, 100)]]
    assert np.concatenate(parts).tobytes() == a.tobytes()
    # device pointers (pairs, out, stats on the GPU)
    dp = torch.from_numpy(pairs).cuda()
    dout = torch.zeros(len(pairs), dtype=torch.float64, device="cuda")
    dst = torch.zeros(len(pairs) * geer.STATS_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    geer.er_query_batch_ex(tiny_h, dp, 0.1, out=dout, stats=dst)
    torch.cuda.synchronize()
    assert dout.cpu().numpy().tobytes() == a.tobytes()
    # plain 3-call API
    c = geer.er_query_batch(tiny_h, pairs, 0.1, 0.01)
    assert c.tobytes() == a.tobytes()


def test_edge_cases(geer, tiny, tiny_h):
    g, pairs = tiny
    out, st = geer.er_query_batch_ex(tiny_h, np.zeros((0, 2), np.int32), 0.1)
    assert out.shape == (0,)
    same = np.array([[5, 5], [0, 0]], dtype=np.int32)
    out, st = geer.er_query_batch_ex(tiny_h, same, 0.1, stats=True)
    assert (out == 0.0).all() and (st["ell"] == 0).all()
    with pytest.raises(geer.GeerError) as e:
        geer.er_query_batch(tiny_h, np.array([[0, g.n]], np.int32), 0.1)
    assert e.value.code == geer.ER_EINVAL
    with pytest.raises(geer.GeerError):
        geer.er_query_batch(tiny_h, pairs, -0.1)
    with pytest.raises(geer.GeerError):
        geer.er_query_batch(tiny_h, pairs, 0.1, 1.5)
    # ell = 0 (huge eps): r' = 1/d_s + 1/d_t exactly (R3)
    out, st = geer.er_query_batch_ex(tiny_h, pairs[:10], 50.0, stats=True)
    d = g.degrees()
    assert (st["ell"] == 0).all()
    assert np.array_equal(out, 1.0 / d[pairs[:10, 0]] + 1.0 / d[pairs[:10, 1]])
    # lambda must be set before queries
    h2 = geer.er_graph_create(g.n, g.offsets, g.cols)
    with pytest.raises(geer.GeerError) as e:
        geer.er_query_batch(h2, pairs, 0.1)
    assert e.value.code == geer.ER_ESPECTRAL
    geer.er_graph_destroy(h2)


def test_fig3_integer_spmm(geer):
    import torch
    from pathlib import Path
    gold = {}
    for line in (Path(__file__).parent / "golden" / "fig3_paths.txt").read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            k, *v = line.split()
            gold[k] = [int(x) for x in v]
    g, idx = W.toy_fig3()
    h = geer.er_graph_create(g.n, g.offsets, g.cols, flags=geer.ER_CREATE_SPMM_ONLY)
    X = torch.zeros((g.n, 2), dtype=torch.float64, device="cuda")
    X[idx["s"], 0] = 1.0
    X[idx["t"], 1] = 1.0
    rows_s, rows_t = [], []
    for _ in range(8):
        Y = torch.empty_like(X)
        geer.er_spmm(h, X, Y, normalize=False)
        X = Y
        tot = X.sum(0).cpu().numpy()
        rows_s.append(int(tot[0]))
        rows_t.append(int(tot[1]))
    assert rows_s == gold["path_s"] and rows_t == gold["path_t"]
    with pytest.raises(geer.GeerError) as e:
        geer.er_query_batch(h, [[0, 1]], 0.1)
    assert e.value.code == geer.ER_EBIPARTITE
    geer.er_graph_destroy(h)


def test_spmm_matches_dense_and_series(geer):
    import torch
    g = W.random_small(3, 60, 0.08)
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    X = np.random.default_rng(0).random((g.n, 7))
    Y = torch.empty((g.n, 7), dtype=torch.float64, device="cuda")
    geer.er_spmm(h, torch.from_numpy(X).cuda(), Y)
    assert np.allclose(Y.cpu().numpy(), exact.dense_P(g) @ X, atol=1e-13)
    # oracle's own dense propagation is bit-identical (same CSR-order sums)
    assert np.array_equal(Y.cpu().numpy()[:, 3], oracle.propagate_dense(g, X[:, 3]))
    geer.er_graph_destroy(h)


@pytest.mark.parametrize("n", [5, 10])
def test_complete_graph_series_on_gpu(geer, n):
    g = W.complete(n)
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    geer.er_graph_set_lambda(h, 1.0 / (n - 1))
    out, st = geer.er_query_batch_ex(h, [[0, 1], [2, 4]], 1e-9, force_ell_b=1000, stats=True)
    ell = int(st["ell"][0])
    assert ell >= 4 and (st["ell_f"] == 0).all()
    want = (2 / n) * (1 - (-1 / (n - 1)) ** (ell + 1))
    assert np.abs(out - want).max() < 1e-14
    terms = st["rb_terms"][0][:min(ell, 8)]
    i = np.arange(1, len(terms) + 1)
    # term_i = r_i - r_{i-1} = (2/n) (-1/(n-1))^i (1 + 1/(n-1))
    assert np.allclose(terms, (2 / n) * (-1 / (n - 1)) ** i * (1 + 1 / (n - 1)), rtol=1e-12, atol=1e-16)
    geer.er_graph_destroy(h)


def test_lanczos_lambda(geer, tiny):
    g, _ = tiny
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    lam = geer.er_graph_estimate_lambda(h)
    true = exact.lambda_dense(g)
    assert true - 1e-12 <= lam <= true + 1e-6
    assert geer.er_graph_lambda(h) == lam
    for gg, want in [(W.petersen(), 2 / 3), (W.complete(6), 1 / 5), (W.cycle(9), np.cos(np.pi / 9))]:
        hh = geer.er_graph_create(gg.n, gg.offsets, gg.cols)
        assert abs(geer.er_graph_estimate_lambda(hh) - want) < 1e-6
        geer.er_graph_destroy(hh)
    geer.er_graph_destroy(h)


def _expander_ring(k=4, n=300, p=0.02, seed=3):
    """k random connected non-bipartite graphs joined in a ring by one edge each: the k - 1
    eigenvalues of P below 1 that the ring's bottlenecks create cluster near 1 (and the ring's
    symmetry makes some of them nearly degenerate)."""
    E = []
    for b in range(k):
        gb = W.random_small(seed + b, n, p)
        rows = np.repeat(np.arange(n), gb.degrees())
        E += [(b * n + int(u), b * n + int(v)) for u, v in zip(rows, gb.cols) if u < v]
        E.append((b * n + 5, ((b + 1) % k) * n + 7))
    return W.from_edges(k * n, E, "expander_ring")


def test_lanczos_lambda_clustered_extremes(geer):
    """The device Lanczos (full re-orthogonalisation, both ends converged, explicit residuals)
    returns an upper estimate of lambda on a graph whose extreme eigenvalues are clustered."""
    g = _expander_ring()
    true = exact.lambda_dense(g)
    ev = np.sort(np.abs(np.linalg.eigvalsh(exact.dense_N(g))))[::-1] if hasattr(exact, "dense_N") else None
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        est = geer.er_graph_estimate_lambda(h)
    finally:
        geer.er_graph_destroy(h)
    assert true - 1e-12 <= est <= true + 1e-7, (est, true, ev[:6] if ev is not None else None)


def test_rmat20_lambda_vs_arpack(geer, rmat20):
    # the device estimate is an upper estimate (R12), close to ARPACK; the fixture pins ARPACK's
    # lambda on both sides, so the estimate is taken on a second handle
    g, _, _, _ = rmat20
    ref = W.lambda_of(g)
    assert 0.0 <= g.lam - ref <= 2e-12   # lambda_for rounds ARPACK up to the 1e-12 grid
    h2 = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        est = geer.er_graph_estimate_lambda(h2)
    finally:
        geer.er_graph_destroy(h2)
    assert ref - 1e-12 <= est <= ref + 1e-8   # full re-orthogonalisation + explicit residuals


@pytest.mark.parametrize("kw", [dict(switch_ratio=0.3), dict(reuse_samples=1)])
def test_rmat20_parity_variants(geer, rmat20, kw):
    """SURVEY 8(f)#4 variant knobs at config-1 size (first 2000 queries): GPU = oracle."""
    g, pairs, _, h = rmat20
    sub = np.concatenate([pairs[:1000], pairs[5000:6000]])
    r, st, ro, so = run_both(geer, h, g, sub, 0.1, **kw)
    compare(g, sub, r, st, ro, so)


@pytest.mark.parametrize("eps", [0.5, 0.2, 0.1])
def test_rmat20_parity_full(geer, rmat20, eps):
    g, pairs, _, h = rmat20
    r, st, ro, so = run_both(geer, h, g, pairs, eps)
    compare(g, pairs, r, st, ro, so)
    a, _ = geer.er_query_batch_ex(h, pairs, eps)
    assert a.tobytes() == r.tobytes()


def test_rmat20_parity_eps005_subset(geer, rmat20):
    g, pairs, _, h = rmat20
    sub = pairs[::10]
    r, st, ro, so = run_both(geer, h, g, sub, 0.05, query_index_base=3)
    compare(g, sub, r, st, ro, so)


def test_launch_counter(geer, tiny, tiny_h):
    g, pairs = tiny
    n0 = geer.er_graph_kernel_launches(tiny_h)
    geer.er_query_batch(tiny_h, pairs, 0.1)
    assert geer.er_graph_kernel_launches(tiny_h) > n0


def test_unsorted_rows_parity(geer, tiny):
    # adjacency rows in a random order: walks index rows in input order on both sides (R10);
    # SMM sums differ from the oracle's CSR-order sums only by rounding (R13, 1e-10 relative)
    g0, pairs = tiny
    rng = np.random.default_rng(5)
    cols = g0.cols.copy()
    for v in range(g0.n):
        a, b = g0.offsets[v], g0.offsets[v + 1]
        cols[a:b] = rng.permutation(cols[a:b])
    g = W.Graph(g0.n, g0.offsets.copy(), cols, "tiny_shuffled", g0.lam)
    import os
    for layout in ("", "dord"):   # default walk layout, and the degree-ordered one (row order kept)
        if layout:
            os.environ["GEER_WALK_LAYOUT"] = layout
        try:
            h = geer.er_graph_create(g.n, g.offsets, g.cols)
        finally:
            os.environ.pop("GEER_WALK_LAYOUT", None)
        geer.er_graph_set_lambda(h, g.lam)
        for eps in (0.1, 0.3):
            r, st, ro, so = run_both(geer, h, g, pairs, eps)
            compare(g, pairs, r, st, ro, so, sorted_adj=False)
        geer.er_graph_destroy(h)


@pytest.mark.parametrize("graph", ["tiny", "rmat20"])
def test_walk_layouts_byte_identical(geer, tiny, rmat20, graph):
    # node records + columns (32-bit or 24-bit, 5 per 16-byte chunk), 16-byte arc records, packed
    # 8-byte arc records and the degree-ordered renumbering (24-bit columns + a class tree, y-tables
    # keyed by the new ids) are five encodings of the same CSR: every output bit must agree
    #
    import os
    if graph == "tiny":
        g, pairs = tiny
        pairs = pairs
    else:
        g, pairs, _, _ = rmat20
        pairs = pairs[::20]
    outs = {}
    code = {"cols": 0, "arcs": 1, "packed": 2, "cols24": 3, "dord": 4}
    for lay in ("cols", "cols24", "arcs", "packed", "dord"):
        os.environ["GEER_WALK_LAYOUT"] = lay
        try:
            h = geer.er_graph_create(g.n, g.offsets, g.cols)
        finally:
            del os.environ["GEER_WALK_LAYOUT"]
        assert geer.er_graph_profile_read(h)["walk_layout"] == code[lay]
        geer.er_graph_set_lambda(h, g.lam)
        r, st = geer.er_query_batch_ex(h, pairs, 0.1, stats=True)
        outs[lay] = (r.tobytes(), st.tobytes())
        geer.er_graph_destroy(h)
    assert outs["cols"] == outs["cols24"] == outs["arcs"] == outs["packed"] == outs["dord"]


def test_degree_ordered_layout_budget(geer, rmat20):
    # layout 4's class tables must fit the shared-memory budget: a smaller budget takes a larger
    # block (more padding ids, a different renumbering), a budget nothing fits falls back to the
    # 24-bit columns; every output bit stays the same
    import os
    g, pairs, _, _ = rmat20
    pairs = pairs[::10]
    outs = {}
    for kb, want in (("24", 4), ("8", 4), ("0", 3)):
        os.environ.update({"GEER_WALK_LAYOUT": "dord", "GEER_DORD_SMEM_KB": kb})
        try:
            h = geer.er_graph_create(g.n, g.offsets, g.cols)
        finally:
            del os.environ["GEER_WALK_LAYOUT"], os.environ["GEER_DORD_SMEM_KB"]
        prof = geer.er_graph_profile_read(h)
        assert prof["walk_layout"] == want, (kb, prof["walk_layout"])
        geer.er_graph_set_lambda(h, g.lam)
        r, st = geer.er_query_batch_ex(h, pairs, 0.1, stats=True)
        # ytable_log2 is a diagnostic of the y-table layout, which the rank/hash rule picks from
        # the walk id range (padded under layout 4): every other field must agree
        st = st.copy()
        st["ytable_log2"] = 0
        outs[kb] = (r.tobytes(), st.tobytes(), prof["walk_graph_bytes"])
        geer.er_graph_destroy(h)
    assert outs["24"][:2] == outs["8"][:2] == outs["0"][:2]
    assert outs["8"][2] >= outs["24"][2]   # more padding ids, larger perm tables


def _hub_graph(n=3000, seed=5):
    """Hubs of degree n-1 and 1500 (K9 rows cut into SPMM_SEG = 512 segments) over a sparse
    random graph, plus rows of degree exactly 512 and 513 (the segment boundary)."""
    rng = np.random.default_rng(seed)
    E = [(0, i) for i in range(1, n)] + [(1, int(j)) for j in rng.choice(np.arange(2, n), min(1500, n - 2), replace=False)]
    if n >= 1200:
        E += [(2, int(j)) for j in range(3, 3 + 510)] + [(3, int(j)) for j in range(600, 600 + 510)]
    iu = rng.integers(4, n, 4 * n)
    ju = rng.integers(4, n, 4 * n)
    E += [(int(a), int(b)) for a, b in zip(iu, ju) if a != b]
    return W.from_edges(n, E, "hubs")


def _seg_sum_pull(g, x, normalize, seg=512):
    """K9's documented order (R13): sequential inside segments of 512 neighbours,
    segment sums added in order; equals the plain sequential pull on rows of degree <= 512."""
    y = np.zeros(g.n)
    for v in range(g.n):
        nb = g.neighbors(v)
        acc = 0.0
        for s0 in range(0, len(nb), seg):
            part = 0.0
            for w in nb[s0:s0 + seg]:
                part += x[w]
            acc += part
        y[v] = acc / len(nb) if normalize else acc
    return y


@pytest.mark.parametrize("q", [1, 2, 3, 7, 16, 33, 64, 130, 256])
def test_spmm_k9_every_column(geer, q):
    """K9 (light rows and segmented heavy rows, both vector widths): rows of degree <= 512 are
    bit-identical to the oracle's sequential dense pull (R13); longer rows equal the documented
    segmented order bit for bit and the oracle within 1e-13 relative; for A and P = D^-1 A."""
    import torch
    g = _hub_graph()
    d = g.degrees()
    assert d.max() == g.n - 1 and (d > 512).sum() >= 2 and {512, 513} <= set(d.tolist())
    light = d <= 512
    h = geer.er_graph_create(g.n, g.offsets, g.cols, flags=geer.ER_CREATE_SPMM_ONLY)
    try:
        X = np.random.default_rng(q).random((g.n, q))
        Xd = torch.from_numpy(X).cuda()
        for normalize in (True, False):
            Y = torch.full((g.n, q), np.nan, dtype=torch.float64, device="cuda")
            geer.er_spmm(h, Xd, Y, normalize=normalize)
            Yh = Y.cpu().numpy()
            for c in range(q) if q <= 16 else (0, q // 2, q - 1):
                want = oracle.propagate_dense(g, X[:, c], normalize=normalize)
                assert np.array_equal(Yh[light, c], want[light]), (q, c, normalize)
                assert np.allclose(Yh[~light, c], want[~light], rtol=1e-13, atol=0), (q, c, normalize)
                assert np.array_equal(Yh[~light, c], _seg_sum_pull(g, X[:, c], normalize)[~light])
    finally:
        geer.er_graph_destroy(h)


@pytest.mark.parametrize("q", [2, 6, 16, 64])
def test_spmm_k9_item_pipeline_row_lengths(geer, q):
    """k_spmm_items (q <= 64) hands each sub-warp rows one after another, loading the next row's
    first neighbour ids during the current row's last gather round: rows of every degree 1..60
    (around multiples of the 6 gathers per round), interleaved in id order, bit-identical to the
    oracle's sequential pull, in both the exact and the segmented mode."""
    import torch
    E, nxt = [], 60
    for c in range(60):                     # star centre c: c + 1 leaves, chained to c + 1
        for _ in range(c):
            E.append((c, nxt))
            nxt += 1
        if c + 1 < 60:
            E.append((c, c + 1))
    E += [(0, nxt), (nxt, nxt + 1)]         # degree 2
    g = W.from_edges(nxt + 2, E, "stars")
    assert set(range(1, 61)) <= set(g.degrees().tolist())
    h = geer.er_graph_create(g.n, g.offsets, g.cols, flags=geer.ER_CREATE_SPMM_ONLY)
    try:
        X = np.random.default_rng(40 + q).random((g.n, q))
        Xd = torch.from_numpy(X).cuda()
        for exact_ in (False, True):
            for normalize in (True, False):
                Y = torch.full((g.n, q), np.nan, dtype=torch.float64, device="cuda")
                geer.er_spmm(h, Xd, Y, normalize=normalize, exact=exact_)
                Yh = Y.cpu().numpy()
                for c in range(q) if q <= 16 else (0, 31, q - 1):
                    want = oracle.propagate_dense(g, X[:, c], normalize=normalize)
                    assert np.array_equal(Yh[:, c], want), (q, c, exact_, normalize)
    finally:
        geer.er_graph_destroy(h)


def test_spmm_k9_unaligned_block(geer):
    """A block whose base is only 8-byte aligned takes the scalar path; same bits."""
    import torch
    g = _hub_graph(800, 7)
    h = geer.er_graph_create(g.n, g.offsets, g.cols, flags=geer.ER_CREATE_SPMM_ONLY)
    try:
        q = 4
        X = np.random.default_rng(1).random((g.n, q))
        buf = torch.zeros(g.n * q + 1, dtype=torch.float64, device="cuda")
        Xd = buf[1:].view(g.n, q)
        Xd.copy_(torch.from_numpy(X))
        ybuf = torch.zeros(g.n * q + 1, dtype=torch.float64, device="cuda")
        Y = ybuf[1:].view(g.n, q)
        geer.er_spmm(h, Xd, Y)
        light = g.degrees() <= 512
        for c in range(q):
            want = oracle.propagate_dense(g, X[:, c])
            got = Y.cpu().numpy()[:, c]
            assert np.array_equal(got[light], want[light])
            assert np.allclose(got[~light], want[~light], rtol=1e-13, atol=0)
    finally:
        geer.er_graph_destroy(h)


def test_spmm_k9_rmat20_sampled_columns(geer, rmat20):
    """At BASELINE config 1's full size, in bench.py's launch configuration (q = 16): two
    columns checked against the oracle's pull over all n rows (bit-exact on rows of degree
    <= 512, 1e-13 relative on the segmented hub rows)."""
    import torch
    g, _, _, h = rmat20
    q = 16
    X = np.random.default_rng(3).random((g.n, q))
    Y = torch.empty((g.n, q), dtype=torch.float64, device="cuda")
    geer.er_spmm(h, torch.from_numpy(X).cuda(), Y)
    Yh = Y.cpu().numpy()
    light = g.degrees() <= 512
    for c in (0, 11):
        want = oracle.propagate_dense(g, X[:, c])
        assert np.array_equal(Yh[light, c], want[light])
        assert np.allclose(Yh[~light, c], want[~light], rtol=1e-13, atol=0)


def test_query_ids_partition_reproduces_batch(geer, rmat20):
    """Cost-model partition (dist.partition) with global query ids: every query's result is
    byte-identical to the unsharded batch (RNG keyed by the global index, R10), for host and
    device id arrays; and an id outside [0, 2^32) is rejected."""
    import torch
    from paper_2312_06123_b200.dist import partition, predicted_cost
    g, pairs, _, h = rmat20
    sub = pairs[:2000]
    full, _ = geer.er_query_batch_ex(h, sub, 0.2)
    parts = partition(predicted_cost(sub, g.degrees(), g.lam, 0.2), 3)
    got = np.empty_like(full)
    for r, idx in enumerate(parts):
        if r == 0:
            got[idx] = geer.er_query_batch_ex(h, sub[idx], 0.2, query_ids=idx)[0]
        else:   # device pairs + device ids
            out = torch.zeros(len(idx), dtype=torch.float64, device="cuda")
            geer.er_query_batch_ex(h, torch.from_numpy(np.ascontiguousarray(sub[idx])).cuda(), 0.2, out=out,
                                   query_ids=torch.from_numpy(idx.astype(np.int64)).cuda())
            got[idx] = out.cpu().numpy()
    assert got.tobytes() == full.tobytes()
    with pytest.raises(geer.GeerError):
        geer.er_query_batch_ex(h, sub[:2], 0.2, query_ids=np.array([0, 1 << 32]))


@pytest.mark.parametrize("graph", ["tiny", "rmat20"])
def test_ytable_layouts_and_kernel_variants_byte_identical(graph, tiny, rmat20):
    """The y-table layout (hash / rank bitmap), shared-memory staging of small hash
    tables and the walk-kernel schedule (persistent or not, overlap with the head) change no
    output bit: they are layouts and schedules of the same arithmetic.  Two walk pairs per thread regroup the per-chunk partial
    sums (64 walks per warp instead of 32): walk endpoints stay bit-identical, estimates agree
    to ulps.  Each combination runs in a fresh process (the knobs are read at
    er_graph_create)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); import workloads as W;"
            "import paper_2312_06123_b200 as G;"
            f"g, pairs, _ = W.load_config('{graph}');"
            "h = G.er_graph_create(g.n, g.offsets, g.cols); G.er_graph_set_lambda(h, float(sys.argv[1]));"
            "r, st = G.er_query_batch_ex(h, pairs[:3000], 0.1, stats=True);"
            "sys.stdout.buffer.write(r.tobytes() + st['walk_checksum'].tobytes())")
    g = (tiny if graph == "tiny" else rmat20)[0]
    outs = {}
    for env in ({"GEER_YTABLE": "hash"}, {"GEER_YTABLE": "rank"}, {}, {"GEER_RANK_MAX_KB": "0"},
                {"GEER_WALK_SMEM_KB": "8"}, {"GEER_WALK_SMEM_KB": "24", "GEER_YTABLE": "hash"},
                {"GEER_WALK_TILES": "1"}, {"GEER_WALK_LAYOUT": "arcs"}, {"GEER_WALK_LAYOUT": "cols"},
                {"GEER_WALK_NP": "2"}, {"GEER_WALK_NP": "2", "GEER_WALK_MINB": "3"}, {"GEER_WALK_PERSIST": "0"},
                {"GEER_AMC_OVERLAP": "1"}, {"GEER_WALK_LAYOUT": "dord"},
                {"GEER_WALK_LAYOUT": "dord", "GEER_YTABLE": "rank"}, {"GEER_WALK_LAYOUT": "dord", "GEER_YTABLE": "hash"},
                {"GEER_WALK_LAYOUT": "dord", "GEER_RANK_MAX_KB": "0"}, {"GEER_WALK_LAYOUT": "dord", "GEER_WALK_SMEM_KB": "8"}):
        e = dict(os.environ, **env)
        outs[str(env)] = subprocess.run([sys.executable, "-c", code, repr(g.lam)], env=e, check=True,
                                        capture_output=True, cwd=str(W.Path(__file__).resolve().parents[1])).stdout
    ref = outs["{}"]
    assert len(ref) > 0
    n = len(ref) // 16
    r0, c0 = np.frombuffer(ref[:8 * n], np.float64), np.frombuffer(ref[8 * n:], np.uint64)
    for k, v in outs.items():
        if "GEER_WALK_NP" in k:
            r1, c1 = np.frombuffer(v[:8 * n], np.float64), np.frombuffer(v[8 * n:], np.uint64)
            assert np.array_equal(c1, c0), k
            assert np.abs(r1 - r0).max() <= 1e-12, k
        else:
            assert v == ref, k


def test_smm_series_tiny_is_exact_er(geer, tiny, tiny_h):
    """er_smm_series (K9 passes over the signed vector, SMM-to-ell) at tol = 1e-11 equals the
    exact ER (dense pseudo-inverse, Def. 2.1) within the Thm 3.1 tail; L is Eq. 6's ell at
    eps = tol; s = t gives 0."""
    g, pairs = tiny
    r, L = geer.er_smm_series(tiny_h, pairs, tol=1e-11)
    ex = exact.er_pinv(g, pairs)
    assert np.abs(r - ex).max() <= 2e-11
    d = g.degrees()
    want_L = [oracle.refined_ell(int(d[s]), int(d[t]), 1e-11, g.lam) for s, t in pairs]
    assert np.array_equal(L, want_L)
    r2, _ = geer.er_smm_series(tiny_h, [[5, 5], [0, 1]], tol=1e-11)
    assert r2[0] == 0.0 and abs(r2[1] - exact.er_pinv(g, np.array([[0, 1]]))[0]) <= 2e-11


def test_smm_series_rmat20_vs_oracle_and_geer_accuracy(geer, rmat20):
    """At BASELINE config 1's size: (1) er_smm_series equals the oracle's signed-vector series
    (same L) within 1e-10 relative on sampled queries; (2) the paper's accuracy protocol:
    GEER's eps = 0.1 estimates are within eps of the converged series (tol 1e-8) on 100 random
    pairs + 100 edges (each holds with probability >= 1 - delta, delta = 0.01)."""
    g, pairs, _, h = rmat20
    sub = np.concatenate([pairs[:100], pairs[5000:5100]])
    truth, L = geer.er_smm_series(h, sub, tol=1e-8)
    for j in (0, 7, 100, 150):
        s, t = (int(x) for x in sub[j])
        ref = oracle.series_signed(g, s, t, int(L[j]))
        assert abs(truth[j] - ref) <= 1e-10 * max(1.0, abs(ref)), j
    est, _ = geer.er_query_batch_ex(h, sub, 0.1)
    err = np.abs(est - truth)
    assert np.mean(err <= 0.1) >= 0.99 and err.max() <= 0.2, err.max()


@pytest.mark.parametrize("config,eps,nq", [("lj_full", 0.1, 100), ("orkut_full", 0.1, 100), ("friendster", 0.1, 40)])
def test_full_size_configs_parity_sampled(geer, config, eps, nq):
    """BASELINE configs 2-4 at full size (GPU R-MAT generator: LiveJournal-shaped n ~ 3.2M,
    m ~ 37M; Orkut-shaped n ~ 4M, m ~ 117M; Friendster-shaped n ~ 60M, m ~ 1.8B), in the
    bench's launch configuration: sampled queries -- the first nq random pairs and the first
    nq edges of the query set, each block with its global query index base -- against the
    oracle (decisions, walk checksums exact; |r' - r'_oracle| <= 1e-9), plus the converged
    series (er_smm_series) within eps on a few of them; then the bench's whole per-GPU batch,
    whose first nq results must be the sampled ones bit for bit."""
    g, pairs, _ = W.load_config(config)
    g.lam = W.lambda_for(g)   # preprocessing lambda (torch Lanczos, not the library's), pinned on both sides
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    try:
        geer.er_graph_set_lambda(h, g.lam)
        half = len(pairs) // 2
        for base in (0, half):
            sub = pairs[base:base + nq]
            r, st = geer.er_query_batch_ex(h, sub, eps, 0.01, stats=True, query_index_base=base)
            ro, so = oracle.geer_batch(g, g.lam, sub, eps, delta=0.01, query_index_base=base,
                                       nthreads=8 if g.n > 10_000_000 else 0)
            compare(g, sub, r, st, ro, so)
            ns = 20 if g.nnz < (1 << 30) else 4
            truth, _ = geer.er_smm_series(h, sub[:ns], tol=1e-7)
            assert np.abs(r[:ns] - truth).max() <= eps
            if base == 0:
                r0 = r
        # the bench's own batch (one GPU's query set, all streams and overlaps as timed): its first
        # nq results are the sampled ones bit for bit (global query indices key every walk)
        nbench = {"lj_full": 100_000, "orkut_full": 100_000, "friendster": 125_000}[config]
        big = np.ascontiguousarray(pairs[:nbench])
        rb, _ = geer.er_query_batch_ex(h, big, eps, 0.01)
        assert np.isfinite(rb).all()
        assert rb[:nq].tobytes() == r0.tobytes()
    finally:
        geer.er_graph_destroy(h)


def test_sub_batches_are_byte_identical(geer, rmat20):
    """A batch split into internal sub-batches (GEER_MAX_SUB_BATCH) returns the bytes of the
    single batch: every query keeps its global index (fresh process: the knob is read at
    er_graph_create)."""
    import os
    import subprocess
    import sys
    g = rmat20[0]
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); import workloads as W;"
            "import paper_2312_06123_b200 as G;"
            "g, pairs, _ = W.load_config('rmat20');"
            "h = G.er_graph_create(g.n, g.offsets, g.cols); G.er_graph_set_lambda(h, float(sys.argv[1]));"
            "r, st = G.er_query_batch_ex(h, pairs[:3000], 0.1, stats=True, query_index_base=123);"
            "sys.stdout.buffer.write(r.tobytes() + st.tobytes())")
    outs = []
    for env in ({}, {"GEER_MAX_SUB_BATCH": "700"}):
        outs.append(subprocess.run([sys.executable, "-c", code, repr(g.lam)], env=dict(os.environ, **env),
                                   check=True, capture_output=True,
                                   cwd=str(W.Path(__file__).resolve().parents[1])).stdout)
    assert len(outs[0]) > 0 and outs[0] == outs[1]


def test_split_waves_are_byte_identical(geer, rmat20):
    """SMM waves pushed in chunks of whole queries (GEER_WAVE_PAIRS_MAX, a forced small cap: far
    below a config-1 wave's ~10^7 pairs, so every push wave is split, single oversize queries
    included) return the bytes of the unsplit run, stats included (fresh process: the knob is read
    at er_graph_create)."""
    import os
    import subprocess
    import sys
    g = rmat20[0]
    code = ("import sys, numpy as np; sys.path.insert(0, '.'); import workloads as W;"
            "import paper_2312_06123_b200 as G;"
            "g, pairs, _ = W.load_config('rmat20');"
            "h = G.er_graph_create(g.n, g.offsets, g.cols); G.er_graph_set_lambda(h, float(sys.argv[1]));"
            "sub = np.ascontiguousarray(np.concatenate([pairs[:1500], pairs[5000:6500]]));"
            "r, st = G.er_query_batch_ex(h, sub, 0.05, stats=True, query_index_base=7, smm_mode=1);"
            "sys.stdout.buffer.write(r.tobytes() + st.tobytes())")
    outs = []
    for env in ({}, {"GEER_WAVE_PAIRS_MAX": "50000"}):
        outs.append(subprocess.run([sys.executable, "-c", code, repr(g.lam)], env=dict(os.environ, **env),
                                   check=True, capture_output=True,
                                   cwd=str(W.Path(__file__).resolve().parents[1])).stdout)
    assert len(outs[0]) > 0 and outs[0] == outs[1]


@pytest.mark.parametrize("case", ["range", "selfloop", "dup", "asym", "disconnected", "bipartite", "ok", "unsorted"])
def test_device_validation_matches_host(geer, case):
    """er_graph_create validates on the device (validate.cu); GEER_HOST_VALIDATE=1 forces the host
    validation.  Both give the same code (and message) on sorted-row graphs with one injected fault,
    at a size where the device path does real work; unsorted rows go to the host either way."""
    import os
    g = W.random_small(11, 3000, 0.004)
    off, cols = g.offsets.copy(), g.cols.copy()
    d = g.degrees()
    v = int(np.argmax(d))
    if case == "range":
        cols[off[v] + 1] = g.n + 7
    elif case == "selfloop":
        cols[off[v]] = v          # (row stays sorted only if v is its smallest neighbour: allow either)
        cols[off[v]:off[v + 1]] = np.sort(cols[off[v]:off[v + 1]])
    elif case == "dup":
        cols[off[v] + 1] = cols[off[v]]
    elif case == "asym":
        # drop v from row u (u = v's first neighbour) by replacing it with another absent neighbour
        u = int(cols[off[v]])
        row = cols[off[u]:off[u + 1]]
        cand = [w for w in range(g.n) if w != u and w not in set(row.tolist())]
        row[row == v] = cand[0]
        cols[off[u]:off[u + 1]] = np.sort(row)
    elif case == "disconnected":
        h = W.from_edges(20, [(i, i + 1) for i in range(9)] + [(0, 2)] + [(10 + i, 11 + i) for i in range(9)] + [(10, 12)])
        off, cols = h.offsets, h.cols
    elif case == "bipartite":
        h = W.cycle(2000)
        off, cols = h.offsets, h.cols
    elif case == "unsorted":
        cols[off[v]:off[v + 1]] = cols[off[v]:off[v + 1]][::-1]
    n = len(off) - 1
    res = {}
    for host in ("0", "1"):
        os.environ["GEER_HOST_VALIDATE"] = host
        try:
            try:
                h = geer.er_graph_create(n, off, cols)
                geer.er_graph_destroy(h)
                res[host] = ("ok", "")
            except geer.GeerError as e:
                res[host] = (e.code, str(e))
        finally:
            del os.environ["GEER_HOST_VALIDATE"]
    assert res["0"] == res["1"], res
    want = {"range": geer.ER_EINVAL, "selfloop": geer.ER_ESELFLOOP, "dup": geer.ER_EDUP, "asym": geer.ER_EASYM,
            "disconnected": geer.ER_EDISCONNECTED, "bipartite": geer.ER_EBIPARTITE, "ok": "ok", "unsorted": "ok"}[case]
    assert res["0"][0] == want, res


@pytest.mark.gpu
def test_probe_random_loads(geer):
    # the live ceiling bench.py quotes K6 against: an L2-resident buffer serves random
    # sectors several times faster than a DRAM-resident one; bad arguments fail with ER_EINVAL
    l2 = geer.er_probe_random_loads(48 << 20, 0, 16)
    dram = geer.er_probe_random_loads(256 << 20, 1, 16)
    assert 100.0 < l2 < 1000.0 and 10.0 < dram < 200.0 and l2 > 2.0 * dram, (l2, dram)
    with pytest.raises(geer.GeerError):
        geer.er_probe_random_loads(1024, 0, 1)
    with pytest.raises(geer.GeerError):
        geer.er_probe_random_loads(48 << 20, 2, 1)


@pytest.mark.gpu
def test_enomem_fault_injection_recovers(geer, tiny):
    # GEER_FAULT_ALLOC=N makes the N-th workspace growth after er_graph_create fail like an
    # out-of-memory cudaMalloc: the batch fails with ER_ENOMEM (or succeeds when N is past the last
    # growth), and the same handle then answers the batch bit-identically to an unfaulted run
    import os
    g, pairs = tiny
    h = geer.er_graph_create(g.n, g.offsets, g.cols)
    geer.er_graph_set_lambda(h, g.lam)
    ref = geer.er_query_batch(h, pairs, 0.1, 0.01)
    geer.er_graph_destroy(h)
    failed = 0
    try:
        for n in (1, 2, 3, 5, 8, 13, 21, 34, 55):
            os.environ["GEER_FAULT_ALLOC"] = str(n)
            h = geer.er_graph_create(g.n, g.offsets, g.cols)
            try:
                geer.er_graph_set_lambda(h, g.lam)
                try:
                    geer.er_query_batch(h, pairs, 0.1, 0.01)
                except geer.GeerError as e:
                    assert e.code == geer.ER_ENOMEM, e
                    failed += 1
                r = geer.er_query_batch(h, pairs, 0.1, 0.01)
                assert r.tobytes() == ref.tobytes(), n
            finally:
                geer.er_graph_destroy(h)
    finally:
        os.environ.pop("GEER_FAULT_ALLOC", None)
        h = geer.er_graph_create(g.n, g.offsets, g.cols)   # resets the injection
        geer.er_graph_destroy(h)
    assert failed >= 3
