"""K9 probe: er_spmm on BASELINE config 1's graph at q = 16 and 64 (for ncu captures)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

g, _, _ = W.load_config(sys.argv[1] if len(sys.argv) > 1 else "rmat20", with_lambda=False)
h = G.er_graph_create(g.n, g.offsets, g.cols)
for q in (16, 64):
    X = torch.rand((g.n, q), dtype=torch.float64, device="cuda")
    Y = torch.empty_like(X)
    for _ in range(3):
        G.er_spmm(h, X, Y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        G.er_spmm(h, X, Y)
    e1.record()
    torch.cuda.synchronize()
    print(f"q={q} ms={e0.elapsed_time(e1) / 5:.3f}")
G.er_graph_destroy(h)
