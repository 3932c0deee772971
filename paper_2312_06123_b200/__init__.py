"""B200-native GEER: epsilon-approximate pairwise effective resistance queries.

Thin ctypes binding over ``libgeer.so`` (include/geer.h).  Argument marshalling
only: every step of a query runs in the library's CUDA kernels.  There is no
CPU fallback -- the first call into the library raises if the shared library is
missing or fails to load.  The library is loaded lazily (on the first ABI call or
the first access of ``lib``), so host-only modules of the package (``dist``) import
without it.

Names follow the C ABI: ``er_graph_create``, ``er_query_batch``,
``er_graph_destroy`` (+ ``er_query_batch_ex``, ``er_graph_set_lambda``, ...).
Arrays may be numpy arrays (host) or torch CUDA tensors (device pointers).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
# GEER_LIB: an alternative build of this library (A/B experiments, scripts/build_variant.py)
LIB_PATH = Path(os.environ["GEER_LIB"]).resolve() if os.environ.get("GEER_LIB") else _PKG / "libgeer.so"

ER_OK, ER_EINVAL, ER_ESELFLOOP, ER_EDUP, ER_EASYM, ER_EDISCONNECTED, ER_EBIPARTITE, ER_ESPECTRAL, \
    ER_ENOMEM, ER_ECUDA = range(10)
ER_DEFAULT_SEED = 0x2312061232DEC0DE

ERROR_NAMES = {0: "ER_OK", 1: "ER_EINVAL", 2: "ER_ESELFLOOP", 3: "ER_EDUP", 4: "ER_EASYM",
               5: "ER_EDISCONNECTED", 6: "ER_EBIPARTITE", 7: "ER_ESPECTRAL", 8: "ER_ENOMEM", 9: "ER_ECUDA"}

# er_query_stats (include/geer.h), 176 bytes.
STATS_DTYPE = np.dtype([
    ("ell", "<i4"), ("ell_b", "<i4"), ("ell_f", "<i4"), ("batches_run", "<i4"),
    ("eta0", "<i8"), ("walks_total", "<i8"), ("steps_total", "<i8"),
    ("vol_last", "<i8"), ("h_last", "<i8"),
    ("psi", "<f8"), ("r_b", "<f8"), ("r_f", "<f8"), ("f_last", "<f8"), ("sigma2_last", "<f8"),
    ("rb_terms", "<f8", (8,)),
    ("walk_checksum", "<u8"), ("tie_flags", "<u4"), ("ytable_log2", "<u4"),
])

EXPORTED = ["er_graph_create", "er_graph_create_ex", "er_graph_destroy", "er_query_batch", "er_last_error",
            "er_last_error_message", "er_graph_lambda", "er_graph_set_lambda",
            "er_graph_estimate_lambda", "er_graph_num_nodes", "er_graph_num_arcs",
            "er_graph_kernel_launches", "er_opts_default", "er_query_batch_ex", "er_spmm",
            "er_graph_profile", "er_graph_profile_read", "er_smm_series", "er_spmm_ex", "er_probe_random_loads"]


class er_opts(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_int32), ("force_ell_b", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("query_index_base", ctypes.c_int64), ("cuda_stream", ctypes.c_void_p),
                ("pairs_on_device", ctypes.c_int32), ("out_on_device", ctypes.c_int32),
                ("ell_variant", ctypes.c_int32), ("synchronous", ctypes.c_int32), ("pad0", ctypes.c_int32),
                ("query_ids", ctypes.c_void_p), ("switch_ratio", ctypes.c_double), ("reuse_samples", ctypes.c_int32),
                ("smm_mode", ctypes.c_int32)]


class er_profile(ctypes.Structure):
    _fields_ = [("smm_ms", ctypes.c_double), ("walk_ms", ctypes.c_double), ("amc_other_ms", ctypes.c_double),
                ("walk_launches", ctypes.c_int64), ("walk_steps", ctypes.c_int64),
                ("smm_pairs", ctypes.c_int64), ("batches", ctypes.c_int64),
                ("ytable_slots", ctypes.c_int64), ("yrank_records", ctypes.c_int64),
                ("walk_ctas_per_sm", ctypes.c_int64), ("smm_waves", ctypes.c_int64),
                ("smm_dense_waves", ctypes.c_int64), ("smm_dense_cols", ctypes.c_int64),
                ("amc_span_ms", ctypes.c_double), ("walk_graph_bytes", ctypes.c_int64),
                ("walk_layout", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class GeerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    L.er_graph_create.argtypes = [i64, vp, vp]
    L.er_graph_create.restype = vp
    L.er_graph_create_ex.argtypes = [i64, vp, vp, ctypes.c_uint32]
    L.er_graph_create_ex.restype = vp
    L.er_graph_destroy.argtypes = [vp]
    L.er_graph_destroy.restype = None
    L.er_query_batch.argtypes = [vp, vp, i64, dbl, dbl, vp]
    L.er_query_batch.restype = ctypes.c_int
    L.er_query_batch_ex.argtypes = [vp, vp, i64, dbl, dbl, ctypes.POINTER(er_opts), vp, vp]
    L.er_query_batch_ex.restype = ctypes.c_int
    L.er_last_error.restype = ctypes.c_int
    L.er_last_error_message.restype = ctypes.c_char_p
    L.er_graph_lambda.argtypes = [vp, ctypes.POINTER(dbl)]
    L.er_graph_set_lambda.argtypes = [vp, dbl]
    L.er_graph_estimate_lambda.argtypes = [vp, ctypes.c_int, ctypes.POINTER(dbl)]
    for f in ("er_graph_num_nodes", "er_graph_num_arcs", "er_graph_kernel_launches"):
        getattr(L, f).argtypes = [vp]
        getattr(L, f).restype = i64
    L.er_opts_default.argtypes = [ctypes.POINTER(er_opts)]
    L.er_opts_default.restype = None
    L.er_spmm.argtypes = [vp, vp, vp, i32, i32, vp]
    L.er_spmm.restype = ctypes.c_int
    L.er_spmm_ex.argtypes = [vp, vp, vp, i32, i32, vp]
    L.er_spmm_ex.restype = ctypes.c_int
    L.er_probe_random_loads.argtypes = [i64, i32, i32, ctypes.POINTER(dbl)]
    L.er_probe_random_loads.restype = ctypes.c_int
    L.er_smm_series.argtypes = [vp, vp, i64, dbl, i32, vp, vp]
    L.er_smm_series.restype = ctypes.c_int
    L.er_graph_profile.argtypes = [vp, ctypes.c_int]
    L.er_graph_profile_read.argtypes = [vp, ctypes.POINTER(er_profile)]
    return L


_lib = None


def _get():
    """The loaded libgeer.so (loaded on first use; raises ImportError if it is missing)."""
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def __getattr__(name):   # PEP 562: ``paper_2312_06123_b200.lib`` loads the library lazily
    if name == "lib":
        return _get()
    raise AttributeError(name)


def _raise(rc: int):
    if rc != ER_OK:
        raise GeerError(rc, _get().er_last_error_message().decode())


def _ptr(a):
    """(pointer, on_device) of a numpy array or torch tensor."""
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr()), bool(a.is_cuda)
    return a.ctypes.data_as(ctypes.c_void_p), False


def er_last_error() -> int:
    return int(_get().er_last_error())


def er_last_error_message() -> str:
    return _get().er_last_error_message().decode()


ER_CREATE_SPMM_ONLY = 1


def er_graph_create(n: int, offsets, cols, flags: int = 0) -> int:
    """Copy a host CSR (int64 offsets[n+1], int32 cols) to the current CUDA device."""
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    col = np.ascontiguousarray(cols, dtype=np.int32)
    h = _get().er_graph_create_ex(int(n), off.ctypes.data_as(ctypes.c_void_p), col.ctypes.data_as(ctypes.c_void_p),
                               int(flags))
    if not h:
        _raise(er_last_error() or ER_ECUDA)
    return h


def er_graph_destroy(g) -> None:
    _get().er_graph_destroy(g)


def er_graph_set_lambda(g, lam: float) -> None:
    _raise(_get().er_graph_set_lambda(g, float(lam)))


def er_graph_lambda(g) -> float:
    out = ctypes.c_double(0.0)
    _raise(_get().er_graph_lambda(g, ctypes.byref(out)))
    return out.value


def er_graph_estimate_lambda(g, iters: int = 0) -> float:
    out = ctypes.c_double(0.0)
    _raise(_get().er_graph_estimate_lambda(g, int(iters), ctypes.byref(out)))
    return out.value


def er_graph_kernel_launches(g) -> int:
    return int(_get().er_graph_kernel_launches(g))


def er_probe_random_loads(nbytes: int, flavour: int, iters: int = 64) -> float:
    """10^9 random 8-byte loads per second on the current device (include/geer.h)."""
    out = ctypes.c_double()
    _raise(_get().er_probe_random_loads(int(nbytes), int(flavour), int(iters), ctypes.byref(out)))
    return out.value


def er_graph_num_nodes(g) -> int:
    return int(_get().er_graph_num_nodes(g))


def er_graph_num_arcs(g) -> int:
    return int(_get().er_graph_num_arcs(g))


def er_opts_default() -> er_opts:
    o = er_opts()
    _get().er_opts_default(ctypes.byref(o))
    return o


def er_query_batch(g, pairs, eps: float, p_fail: float = 0.01):
    """Host arrays in, host array out (synchronous)."""
    p = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
    k = p.shape[0]
    out = np.zeros(k, dtype=np.float64)
    _raise(_get().er_query_batch(g, p.ctypes.data_as(ctypes.c_void_p), k, float(eps), float(p_fail),
                              out.ctypes.data_as(ctypes.c_void_p)))
    return out


def er_query_batch_ex(g, pairs, eps: float, p_fail: float = 0.01, *, out=None, stats=None,
                      tau: int = 5, seed: int = ER_DEFAULT_SEED, query_index_base: int = 0,
                      force_ell_b: int = -1, ell_variant: int = 0, stream=None, synchronous: bool = True,
                      k: int | None = None, query_ids=None, switch_ratio: float = 1.0, reuse_samples: bool = False,
                      smm_mode: int = 0):
    """Extended query.  ``pairs``/``out``/``stats`` are numpy arrays (host) or torch CUDA
    tensors (device); ``out``/``stats`` are allocated on the host when None.
    ``stats=True`` allocates a host STATS_DTYPE array.  Returns (out, stats)."""
    if hasattr(pairs, "data_ptr"):
        pp, pdev = _ptr(pairs)
        kk = int(pairs.numel() // 2) if k is None else k
    else:
        pairs = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
        pp, pdev = _ptr(pairs)
        kk = pairs.shape[0] if k is None else k
    if out is None:
        out = np.zeros(kk, dtype=np.float64)
    if stats is True:
        stats = np.zeros(kk, dtype=STATS_DTYPE)
    op, odev = _ptr(out)
    sp = None
    if stats is not None and stats is not False:
        sp, sdev = _ptr(stats)
        if sdev != odev:
            raise ValueError("out and stats must both be host or both be device arrays")
    else:
        stats = None
    o = er_opts_default()
    o.tau = tau
    o.force_ell_b = force_ell_b
    o.seed = seed & 0xFFFFFFFFFFFFFFFF
    o.query_index_base = query_index_base
    o.pairs_on_device = int(pdev)
    o.out_on_device = int(odev)
    o.ell_variant = ell_variant
    o.synchronous = int(synchronous)
    o.switch_ratio = float(switch_ratio)
    o.reuse_samples = int(bool(reuse_samples))
    o.smm_mode = int(smm_mode)
    if query_ids is not None:
        if hasattr(query_ids, "data_ptr"):
            if bool(query_ids.is_cuda) != bool(pdev):
                raise ValueError("query_ids must live where pairs live (host or device)")
            o.query_ids = ctypes.c_void_p(query_ids.data_ptr())
        else:
            if pdev:
                raise ValueError("query_ids must live where pairs live (host or device)")
            query_ids = np.ascontiguousarray(query_ids, dtype=np.int64)
            if query_ids.shape[0] != kk:
                raise ValueError("query_ids needs one entry per query")
            o.query_ids = query_ids.ctypes.data_as(ctypes.c_void_p)
    if stream is not None:
        o.cuda_stream = _stream_handle(stream)
    _raise(_get().er_query_batch_ex(g, pp, kk, float(eps), float(p_fail), ctypes.byref(o), op, sp))
    return out, stats


def _stream_handle(stream):
    """cudaStream_t for the C ABI: torch streams, raw handles; torch's legacy default stream
    (handle 0) is passed as cudaStreamLegacy (0x1), because NULL means the handle's own stream."""
    if stream is None:
        return None
    h = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return ctypes.c_void_p(h if h else 1)


ER_SPMM_NORMALIZE = 1
ER_SPMM_EXACT = 2
SMM_AUTO, SMM_FRONTIER, SMM_DENSE = 0, 1, 2   # er_opts.smm_mode


def er_spmm(g, X, Y, normalize: bool = True, stream=None, exact: bool = False) -> None:
    """Y = P X (or A X) for row-major n x q device tensors (float64).  ``exact``: every row
    summed sequentially in CSR order (er_spmm_ex with ER_SPMM_EXACT)."""
    q = 1 if X.dim() == 1 else int(X.shape[1])
    if stream is None:   # order with torch's work on the tensors (their producers and readers)
        import torch
        stream = torch.cuda.current_stream(X.device)
    s = _stream_handle(stream)
    if exact:
        flags = (ER_SPMM_NORMALIZE if normalize else 0) | ER_SPMM_EXACT
        _raise(_get().er_spmm_ex(g, ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Y.data_ptr()), q, flags, s))
    else:
        _raise(_get().er_spmm(g, ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(Y.data_ptr()), q, int(normalize), s))


def er_smm_series(g, pairs, tol: float = 1e-10, max_iters: int = 100000):
    """Deterministic series r_L(s,t) truncated at Thm 3.1's tail bound <= tol (SMM-to-ell /
    ground truth, include/geer.h).  Host arrays in/out.  Returns (r, L)."""
    p = np.ascontiguousarray(np.asarray(pairs, dtype=np.int32).reshape(-1, 2))
    k = p.shape[0]
    out = np.zeros(k, dtype=np.float64)
    ells = np.zeros(k, dtype=np.int32)
    _raise(_get().er_smm_series(g, p.ctypes.data_as(ctypes.c_void_p), k, float(tol), int(max_iters),
                             out.ctypes.data_as(ctypes.c_void_p), ells.ctypes.data_as(ctypes.c_void_p)))
    return out, ells


def er_graph_profile(g, enable: bool = True) -> None:
    _raise(_get().er_graph_profile(g, int(enable)))


def er_graph_profile_read(g) -> dict:
    p = er_profile()
    _raise(_get().er_graph_profile_read(g, ctypes.byref(p)))
    return {f: getattr(p, f) for f, _ in er_profile._fields_}


class Graph:
    """RAII wrapper: ``with Graph(n, offsets, cols, lam) as g: g.query(pairs, eps)``."""

    def __init__(self, n, offsets, cols, lam: float | None = None):
        self.h = er_graph_create(n, offsets, cols)
        self.n = int(n)
        if lam is not None:
            er_graph_set_lambda(self.h, lam)

    def query(self, pairs, eps, p_fail=0.01, **kw):
        return er_query_batch_ex(self.h, pairs, eps, p_fail, **kw)

    def close(self):
        if self.h:
            er_graph_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
