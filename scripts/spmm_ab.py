"""K9 A/B: er_spmm on one config at q = 16 / 64 with the L2 flushed before each call (bench.py's
K9 leg), for the library named by GEER_LIB; one JSON line."""
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "lj_full"
g, _, _ = W.load_config(cfg, with_lambda=False)
h = G.er_graph_create(g.n, g.offsets, g.cols)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"lib": os.environ.get("GEER_LIB", "in-tree"), "config": cfg}
for q in (16, 64):
    X = torch.rand((g.n, q), dtype=torch.float64, device="cuda",
                   generator=torch.Generator(device="cuda").manual_seed(q))   # same X for every variant
    Y = torch.empty_like(X)
    ts = []
    for i in range(8):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        G.er_spmm(h, X, Y)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    byts = 8 * (g.n + 1) + 4 * g.nnz + 8 * q * g.nnz + 8 * q * g.n
    ms = statistics.median(ts)
    out[f"q{q}"] = {"ms": ms, "alg_gbs": byts / ms / 1e6, "checksum": float(Y.sum())}
    del X, Y
G.er_graph_destroy(h)
print(json.dumps(out))
