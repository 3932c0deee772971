"""CPU oracle for the GEER query pipeline (arXiv 2312.06123).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_2312_06123_b200``) never imports it, and the
two share no code, header, table or helper.

Two parts:

* ``oracle.exact``: exact effective resistance by the dense Moore-Penrose
  pseudo-inverse of ``L = D - A`` (Def. 2.1 / Eq. 1), plus
  dense spectral helpers.  Pinned by closed forms in ``tests/test_oracle_exact.py``.
* this module: a ctypes binding to ``geer_oracle.c`` (plain C, OpenMP over
  queries), the step-by-step GEER / AMC / SMM estimator of Alg. 1-3.  Pinned by
  the SPEC hand values, Fig. 3's #path rows, Philox known-answer vectors, dense
  matrix powers and the paper's invariants in ``tests/test_oracle_geer.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "geer_oracle.c"
_LIB_PATH = _HERE / "liboracle.so"

STATS_DTYPE = np.dtype([
    ("ell", "<i4"), ("ell_b", "<i4"), ("ell_f", "<i4"), ("batches_run", "<i4"),
    ("eta0", "<i8"), ("walks_total", "<i8"), ("steps_total", "<i8"),
    ("vol_last", "<i8"), ("h_last", "<i8"),
    ("psi", "<f8"), ("r_b", "<f8"), ("r_f", "<f8"), ("f_last", "<f8"), ("sigma2_last", "<f8"),
    ("rb_terms", "<f8", (8,)),
    ("walk_checksum", "<u8"), ("tie_flags", "<u4"), ("pad", "<u4"),
])


class _Opts(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_int), ("seed", ctypes.c_uint64),
                ("query_index_base", ctypes.c_int64), ("force_ell_b", ctypes.c_int),
                ("ell_variant", ctypes.c_int), ("switch_ratio", ctypes.c_double), ("reuse_samples", ctypes.c_int)]


DEFAULT_SEED = 0x2312061232DEC0DE  # same documented default as the library (R10)


def build(force: bool = False) -> Path:
    """Compile geer_oracle.c into liboracle.so (gcc, no FMA contraction)."""
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB_PATH.with_suffix(".so.tmp%d" % os.getpid())
        subprocess.check_call([
            "gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
            "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        P = ctypes.POINTER
        i64, i32, u32, u64, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double
        vp = ctypes.c_void_p
        L.oracle_philox4x32_10.argtypes = [vp, vp, vp]
        L.oracle_walk_hash.argtypes = [u32, u32, u32, u64, i32]
        L.oracle_walk_hash.restype = u64
        L.oracle_refined_ell.argtypes = [i64, i64, dbl, dbl]
        L.oracle_refined_ell.restype = i64
        L.oracle_peng_ell.argtypes = [dbl, dbl]
        L.oracle_peng_ell.restype = i64
        L.oracle_psi.argtypes = [i64, dbl, dbl, dbl, dbl, i64, i64]
        L.oracle_psi.restype = dbl
        L.oracle_eta_star.argtypes = [dbl, dbl, dbl, ctypes.c_int]
        L.oracle_eta_star.restype = dbl
        L.oracle_eta0.argtypes = [dbl, ctypes.c_int]
        L.oracle_eta0.restype = i64
        L.oracle_h.argtypes = [i64, ctypes.c_int]
        L.oracle_h.restype = i64
        L.oracle_bernstein_f.argtypes = [dbl, dbl, dbl, dbl]
        L.oracle_bernstein_f.restype = dbl
        L.oracle_propagate_dense.argtypes = [i64, vp, vp, vp, vp, ctypes.c_int]
        L.oracle_walk.argtypes = [vp, vp, vp, i32, i64, u64, u32, u32, u32, u64, vp, vp]
        L.oracle_walk.restype = i32
        L.oracle_amc_samples.argtypes = [i64, vp, vp, i32, i32, vp, vp, i64, u64, u32, u32, i64, vp]
        L.oracle_geer_batch.argtypes = [i64, vp, vp, dbl, vp, i64, dbl, dbl, P(_Opts), ctypes.c_int, vp, vp]
        L.oracle_geer_batch.restype = ctypes.c_int
        L.oracle_smm.argtypes = [i64, vp, vp, i32, i32, i64, vp, vp, vp]
        L.oracle_smm.restype = dbl
        L.oracle_sizeof_stats.restype = ctypes.c_int
        L.oracle_max_threads.restype = ctypes.c_int
        assert L.oracle_sizeof_stats() == STATS_DTYPE.itemsize, "stats layout mismatch"
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _csr(g):
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    cols = np.ascontiguousarray(g.cols, dtype=np.int32)
    return off, cols


# ---------------------------------------------------------------- closed forms
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def walk_hash(q, b, side, k, endpoint) -> int:
    return int(lib().oracle_walk_hash(q, b, side, k, endpoint))


def refined_ell(ds, dt, eps, lam) -> int:
    return int(lib().oracle_refined_ell(ds, dt, eps, lam))


def peng_ell(eps, lam) -> int:
    return int(lib().oracle_peng_ell(eps, lam))


def psi(lf, max1s, max2s, max1t, max2t, ds, dt) -> float:
    return float(lib().oracle_psi(lf, max1s, max2s, max1t, max2t, ds, dt))


def eta_star(psi_, eps, delta, tau) -> float:
    return float(lib().oracle_eta_star(psi_, eps, delta, tau))


def eta0(eta_star_, tau) -> int:
    return int(lib().oracle_eta0(eta_star_, tau))


def h_budget(eta0_, tau) -> int:
    return int(lib().oracle_h(eta0_, tau))


def bernstein_f(n, var, psi_, d) -> float:
    return float(lib().oracle_bernstein_f(n, var, psi_, d))


# ---------------------------------------------------------------- propagation
def propagate_dense(g, x, normalize=True) -> np.ndarray:
    off, cols = _csr(g)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(g.n, dtype=np.float64)
    lib().oracle_propagate_dense(g.n, _p(off), _p(cols), _p(x), _p(y), 1 if normalize else 0)
    return y


def walk_counts(g, origin, max_len) -> list[int]:
    """#path(origin) for lengths 1..max_len = sum_v (A^i e_origin)(v), by the same
    propagation routine run with A in place of P (Fig. 3)."""
    x = np.zeros(g.n)
    x[origin] = 1.0
    out = []
    for _ in range(max_len):
        x = propagate_dense(g, x, normalize=False)
        out.append(int(round(x.sum())))
    return out


def smm(g, s, t, ell_b):
    off, cols = _csr(g)
    terms = np.zeros(max(ell_b, 1))
    xs = np.zeros(g.n)
    xt = np.zeros(g.n)
    rb = lib().oracle_smm(g.n, _p(off), _p(cols), s, t, ell_b, _p(terms), _p(xs), _p(xt))
    return float(rb), terms[:ell_b], xs, xt


def series_signed(g, s, t, L) -> float:
    """Eq. 4's r_L(s,t) in the single signed-vector form (SURVEY 8(c) reading 1):
    y_0 = e_s/d_s - e_t/d_t, y_{i+1} = P y_i, r_L = sum_{i=0..L} (y_i(s) - y_i(t)),
    each P step the oracle's sequential dense pull."""
    d = np.diff(np.asarray(g.offsets))
    if s == t:
        return 0.0
    y = np.zeros(g.n)
    y[s] = 1.0 / d[s]
    y[t] = -1.0 / d[t]
    total = 0.0
    for i in range(L + 1):
        total += y[s] - y[t]
        if i < L:
            y = propagate_dense(g, y)
    return float(total)


def walk(g, start, lf, seed=DEFAULT_SEED, q=0, b=0, side=0, k=0, y=None):
    off, cols = _csr(g)
    trace = np.zeros(max(lf, 1), dtype=np.int32)
    acc = ctypes.c_double(0.0)
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    end = lib().oracle_walk(_p(off), _p(cols), None if yy is None else _p(yy), start, lf,
                            seed, q, b, side, k, ctypes.byref(acc), _p(trace))
    return int(end), trace[:lf].copy(), acc.value


def amc_samples(g, s, t, xs, xt, lf, count, seed=DEFAULT_SEED, q=0, b=0) -> np.ndarray:
    off, cols = _csr(g)
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    xt = np.ascontiguousarray(xt, dtype=np.float64)
    z = np.zeros(count)
    lib().oracle_amc_samples(g.n, _p(off), _p(cols), s, t, _p(xs), _p(xt), lf, seed, q, b, count, _p(z))
    return z


# ---------------------------------------------------------------- GEER batch
def geer_batch(g, lam, pairs, eps, delta=0.01, tau=5, seed=DEFAULT_SEED, query_index_base=0,
               force_ell_b=-1, ell_variant=0, nthreads=0, with_stats=True, switch_ratio=1.0, reuse_samples=0):
    """Alg. 3 (GEER) per query; returns (r, stats) with stats a STATS_DTYPE array."""
    off, cols = _csr(g)
    pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
    k = pairs.shape[0]
    out = np.zeros(k, dtype=np.float64)
    st = np.zeros(k, dtype=STATS_DTYPE) if with_stats else None
    o = _Opts(tau, seed & 0xFFFFFFFFFFFFFFFF, query_index_base, force_ell_b, ell_variant, float(switch_ratio),
              int(reuse_samples))
    rc = lib().oracle_geer_batch(g.n, _p(off), _p(cols), lam, _p(pairs), k, eps, delta,
                                 ctypes.byref(o), nthreads, _p(out), None if st is None else _p(st))
    if rc != 0:
        raise ValueError("oracle_geer_batch: invalid arguments")
    return out, st


def max_threads() -> int:
    return int(lib().oracle_max_threads())
