"""Small end-to-end run for compute-sanitizer memcheck: tiny graph (all options), an R-MAT
subset with both y-table layouts, K9 and the series."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

g, pairs, _ = W.load_config("tiny")
h = G.er_graph_create(g.n, g.offsets, g.cols)
G.er_graph_estimate_lambda(h)
for kw in ({}, {"force_ell_b": 0}, {"reuse_samples": True}, {"switch_ratio": 0.3}, {"tau": 8}):
    G.er_query_batch_ex(h, pairs, 0.1, stats=True, **kw)
G.er_smm_series(h, pairs[:10], tol=1e-8)
X = torch.rand((g.n, 6), dtype=torch.float64, device="cuda")
Y = torch.empty_like(X)
G.er_spmm(h, X, Y)
torch.cuda.synchronize()
G.er_graph_destroy(h)
g = W.rmat(14, 8, seed=5)
p = W.query_pairs(g, 400, seed=6)
h = G.er_graph_create(g.n, g.offsets, g.cols)
G.er_graph_estimate_lambda(h)
r, st = G.er_query_batch_ex(h, p, 0.1, stats=True)
print("ok", float(np.abs(r).max()), int(st["steps_total"].sum()))
G.er_graph_destroy(h)
