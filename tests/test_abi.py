"""CPU-side checks of the C ABI boundary (no compute calls without a GPU).

* libgeer.so loads and exports every function include/geer.h declares;
* the Python binding's struct layouts equal the C layouts (compiled with gcc);
* host-side graph validation returns the documented error codes (ER_EINVAL,
  ER_ESELFLOOP, ER_EDUP, ER_EASYM, ER_EDISCONNECTED, ER_EBIPARTITE) before any
  device work, and argument errors are reported for NULL handles.
"""
import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "geer.h"


@pytest.fixture(scope="module")
def G():
    import importlib.util
    spec = importlib.util.spec_from_file_location("geer_build", ROOT / "paper_2312_06123_b200" / "build.py")
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    m.build()
    import paper_2312_06123_b200 as G
    return G


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(er_[a-z_]+)\s*\(", text)))


def test_exports_every_declared_symbol(G):
    decl = declared_functions()
    assert "er_graph_create" in decl and "er_query_batch" in decl and "er_graph_destroy" in decl
    out = subprocess.run(["nm", "-D", "--defined-only", str(G.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (er_[a-z_]+)", out))
    assert set(decl) <= exported, set(decl) - exported
    assert set(decl) == set(G.EXPORTED)
    for name in decl:
        getattr(G.lib, name)


def test_struct_layouts_match_c(G, tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(r'''
#include <stddef.h>
#include <stdio.h>
#include "geer.h"
#define O(T, f) printf(#f " %zu\n", offsetof(T, f))
int main(void) {
  printf("stats %zu\n", sizeof(er_query_stats));
  O(er_query_stats, eta0); O(er_query_stats, psi); O(er_query_stats, rb_terms);
  O(er_query_stats, walk_checksum); O(er_query_stats, tie_flags);
  printf("opts %zu\n", sizeof(er_opts));
  O(er_opts, seed); O(er_opts, query_index_base); O(er_opts, cuda_stream);
  O(er_opts, pairs_on_device); O(er_opts, synchronous); O(er_opts, query_ids);
  O(er_opts, switch_ratio); O(er_opts, reuse_samples); O(er_opts, smm_mode);
  printf("profile %zu\n", sizeof(er_profile));
  O(er_profile, walk_ctas_per_sm); O(er_profile, smm_dense_waves); O(er_profile, walk_graph_bytes);
  O(er_profile, walk_layout);
  return 0;
}''')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", str(ROOT / "include"), "-o", str(exe), str(src)])
    vals = dict(line.split() for line in subprocess.check_output([str(exe)], text=True).splitlines())
    vals = {k: int(v) for k, v in vals.items()}
    d = G.STATS_DTYPE
    assert vals["stats"] == d.itemsize
    for f in ("eta0", "psi", "rb_terms", "walk_checksum", "tie_flags"):
        assert vals[f] == d.fields[f][1], f
    o = G.er_opts
    assert vals["opts"] == ctypes.sizeof(o)
    for f in ("seed", "query_index_base", "cuda_stream", "pairs_on_device", "synchronous", "query_ids",
              "switch_ratio", "reuse_samples", "smm_mode"):
        assert vals[f] == getattr(o, f).offset, f
    assert vals["profile"] == ctypes.sizeof(G.er_profile)
    for f in ("walk_ctas_per_sm", "smm_dense_waves", "walk_graph_bytes", "walk_layout"):
        assert vals[f] == getattr(G.er_profile, f).offset, f


def test_defaults(G):
    o = G.er_opts_default()
    assert o.tau == 5 and o.force_ell_b == -1 and o.seed == G.ER_DEFAULT_SEED and o.synchronous == 1
    assert not o.query_ids
    text = HEADER.read_text()
    assert "0x%XULL" % G.ER_DEFAULT_SEED in text


def _expect(G, code, n, off, cols):
    with pytest.raises(G.GeerError) as e:
        G.er_graph_create(n, off, cols)
    assert e.value.code == code, str(e.value)
    assert G.er_last_error() == code


def test_validation_error_codes(G):
    import workloads as W
    _expect(G, G.ER_EINVAL, 1, [0, 0], [])
    _expect(G, G.ER_EINVAL, 3, [0, 2, 1, 2], [1, 2])                      # non-monotone offsets
    _expect(G, G.ER_EINVAL, 3, [0, 1, 2, 3], [1, 5, 0])                   # col out of range
    _expect(G, G.ER_ESELFLOOP, 3, [0, 2, 3, 4], [0, 1, 0, 0])
    _expect(G, G.ER_EDUP, 3, [0, 3, 5, 7], [1, 2, 1, 0, 2, 0, 1])
    _expect(G, G.ER_EASYM, 3, [0, 2, 3, 4], [1, 2, 0, 1])
    two = W.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    _expect(G, G.ER_EDISCONNECTED, two.n, two.offsets, two.cols)
    c4 = W.cycle(4)
    _expect(G, G.ER_EBIPARTITE, c4.n, c4.offsets, c4.cols)
    g, _ = W.toy_fig3()
    _expect(G, G.ER_EBIPARTITE, g.n, g.offsets, g.cols)


def test_null_handle_errors(G):
    out = np.zeros(1)
    p = np.zeros(2, dtype=np.int32)
    rc = G.lib.er_query_batch(None, p.ctypes.data_as(ctypes.c_void_p), 1, 0.1, 0.01, out.ctypes.data_as(ctypes.c_void_p))
    assert rc == G.ER_EINVAL
    assert G.lib.er_graph_set_lambda(None, 0.5) == G.ER_EINVAL
    assert G.lib.er_graph_kernel_launches(None) == -1
    G.lib.er_graph_destroy(None)  # NULL-safe
    r = np.zeros(1)
    assert G.lib.er_smm_series(None, p.ctypes.data_as(ctypes.c_void_p), 1, 1e-8, 10,
                               r.ctypes.data_as(ctypes.c_void_p), None) == G.ER_EINVAL
    assert G.lib.er_spmm(None, None, None, 4, 1, None) == G.ER_EINVAL
    assert G.lib.er_spmm_ex(None, None, None, 4, G.ER_SPMM_EXACT, None) == G.ER_EINVAL
    assert G.lib.er_graph_estimate_lambda(None, 0, None) == G.ER_EINVAL
    assert G.er_last_error() == G.ER_EINVAL and "NULL" in G.er_last_error_message()


def test_opts_validation_without_device(G):
    """Option checks happen before any device work (a NULL graph is reported first; the
    option ranges are covered on the GPU by the parity tests)."""
    o = G.er_opts_default()
    assert o.switch_ratio == 1.0 and o.reuse_samples == 0 and not o.query_ids and o.smm_mode == G.SMM_AUTO
