"""Walk steps per AMC batch of bench.py's rank-0 query set (the units K6 processes per launch):
steps_b = sum over queries still sampling in batch b of 2 * (eta0 << b) * ell_f.  Used to turn an
ncu capture of one K6 launch (batch b of a step) into per-step bytes / sectors."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "lj_full"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
g, _, _ = W.load_config(config)
g.lam = W.lambda_for(g)


class A:
    pass


a = A()
a.config, a.queries = config, bench.QUERIES_PER_GPU[config]
pairs, lo = bench.rank_pairs(g, a, 0)
h = G.er_graph_create(g.n, g.offsets, g.cols)
G.er_graph_set_lambda(h, g.lam)
_, st = G.er_query_batch_ex(h, pairs, eps, 0.01, stats=True, query_index_base=lo)
out = {"config": config, "eps": eps, "lambda": g.lam, "queries": len(pairs)}
for b in range(5):
    m = st["batches_run"] > b
    out[f"batch{b}_steps"] = int((2 * (st["eta0"][m].astype(np.int64) << b) * st["ell_f"][m]).sum())
out["steps_total"] = int(st["steps_total"].sum())
print(json.dumps(out))
G.er_graph_destroy(h)
