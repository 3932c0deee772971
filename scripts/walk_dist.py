"""Distribution of AMC walk steps over y-table sizes (config 1, 10k queries, eps = 0.1)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

g, pairs, _ = W.load_config("rmat20", with_lambda=False)
h = G.er_graph_create(g.n, g.offsets, g.cols)
G.er_graph_estimate_lambda(h)
eps = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
r, st = G.er_query_batch_ex(h, pairs, eps, 0.01, stats=True)
lg = st["ytable_log2"].astype(int)
steps = st["steps_total"].astype(float)
tot = steps.sum()
print(f"eps={eps} total steps {tot:.3e}, queries with AMC {np.sum(lg > 0)}")
for L in sorted(set(lg.tolist())):
    m = lg == L
    print(f"log2cap={L:2d} queries={m.sum():6d} steps={steps[m].sum():.3e} ({100 * steps[m].sum() / tot:5.1f}%) "
          f"ell_f mean={st['ell_f'][m].mean():.1f} walks mean={st['walks_total'][m].mean():.0f}")
half = len(pairs) // 2
print("random-pair share of steps", steps[:half].sum() / tot)
