"""One SMM-mode case for a kernel launch list: python scripts/dense_one.py K EPS MODE (rmat20)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

k, eps, mode = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
g, pairs, _ = W.load_config("rmat20", with_lambda=False)
h = G.er_graph_create(g.n, g.offsets, g.cols)
G.er_graph_estimate_lambda(h)
sub = np.ascontiguousarray(pairs[:k])
for _ in range(2):
    G.er_query_batch_ex(h, sub, eps, smm_mode=mode)
print("MARK", G.er_graph_kernel_launches(h), flush=True)
G.er_query_batch_ex(h, sub, eps, smm_mode=mode)
print("END", G.er_graph_kernel_launches(h), flush=True)
G.er_graph_destroy(h)
