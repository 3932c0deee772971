"""SMM head: push (frontier) vs dense pull (K9) timing per mode, to calibrate the per-wave cost
model (R25).  Prints one JSON line per (config, k, eps, mode)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_06123_b200 as G  # noqa: E402
import workloads as W  # noqa: E402


def main():
    for cfg, ks, epss in (("tiny", (100,), (0.1, 0.05)), ("rmat20", (8, 32, 128, 1000, 10000), (0.1, 0.05))):
        g, pairs, _ = W.load_config(cfg, with_lambda=False)
        h = G.er_graph_create(g.n, g.offsets, g.cols)
        G.er_graph_estimate_lambda(h)
        cases = [(k, eps, -1) for k in ks for eps in epss]
        if cfg == "rmat20":
            cases += [(8, 0.05, 6), (32, 0.05, 6)]
        for k, eps, feb in cases:
            sub = np.ascontiguousarray(pairs[:k])
            if True:
                ref = None
                for mode in (1, 2, 0):
                    G.er_query_batch_ex(h, sub, eps, smm_mode=mode, force_ell_b=feb)   # warm
                    G.er_graph_profile(h, True)
                    reps = 5
                    for _ in range(reps):
                        r, _ = G.er_query_batch_ex(h, sub, eps, smm_mode=mode, force_ell_b=feb)
                    p = G.er_graph_profile_read(h)
                    G.er_graph_profile(h, False)
                    same = None
                    if ref is None:
                        ref = r.tobytes()
                    else:
                        same = r.tobytes() == ref
                    print(json.dumps(dict(cfg=cfg, k=k, eps=eps, force_ell_b=feb, mode=mode, smm_ms=p["smm_ms"] / reps,
                                          walk_ms=p["walk_ms"] / reps, pairs=p["smm_pairs"] // reps,
                                          waves=p["smm_waves"] // reps, dense=p["smm_dense_waves"] // reps, cols=p["smm_dense_cols"] // reps,
                                          same=same)), flush=True)
        G.er_graph_destroy(h)


if __name__ == "__main__":
    main()
