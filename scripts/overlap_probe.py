"""Experiment (profiles/exp_overlap_r02.jsonl; the second set ran with an experiment build whose
K6 grid took 75 % of the resident-CTA slots): would overlapping one sub-batch's SMM head with another's walks pay?  Two graph
handles (own workspaces and streams) answer the two halves of the graded query set, sequentially
and from two host threads (ctypes releases the GIL), with the second thread started `delay` ms
later.  Prints one JSON line per mode; results must be bit-identical to the sequential run."""
import json
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "lj_full"
g, _, _ = W.load_config(cfg)
g.lam = W.lambda_for(g)
nq = 100_000 if cfg != "rmat20" else 10_000
pairs = np.ascontiguousarray(W.query_pairs(g, nq, seed=W.CONFIGS[cfg][1]["seed"] + 1))
A, B = pairs[: nq // 2], pairs[nq // 2:]
hs = []
for _ in range(2):
    h = G.er_graph_create(g.n, g.offsets, g.cols)
    G.er_graph_set_lambda(h, g.lam)
    hs.append(h)
opts = [dict(query_index_base=0), dict(query_index_base=nq // 2)]


def run(h, P, o, out):
    out.append(G.er_query_batch_ex(h, P, 0.1, 0.01, **o)[0])


for h in hs:   # warm-up
    G.er_query_batch_ex(h, A, 0.1, 0.01, query_index_base=0)
torch.cuda.synchronize()
ref = []
t0 = time.perf_counter()
run(hs[0], A, opts[0], ref)
run(hs[0], B, opts[1], ref)
t_seq = time.perf_counter() - t0
print(json.dumps({"mode": "sequential", "ms": t_seq * 1e3}), flush=True)
for delay in (0.0, 0.02, 0.04, 0.06):
    oa, ob = [], []
    t0 = time.perf_counter()
    ta = threading.Thread(target=run, args=(hs[0], A, opts[0], oa))
    tb = threading.Thread(target=run, args=(hs[1], B, opts[1], ob))
    ta.start()
    time.sleep(delay)
    tb.start()
    ta.join()
    tb.join()
    t = time.perf_counter() - t0
    same = oa[0].tobytes() == ref[0].tobytes() and ob[0].tobytes() == ref[1].tobytes()
    print(json.dumps({"mode": "two threads", "delay_ms": delay * 1e3, "ms": t * 1e3, "vs_seq": t / t_seq,
                      "bit_identical": same, "slot_frac": os.environ.get("GEER_WALK_SLOT_FRAC", "1.0")}), flush=True)
for h in hs:
    G.er_graph_destroy(h)
