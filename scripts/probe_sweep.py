"""er_probe_random_loads by buffer size and load flavour (-> profiles/probe_sweep_r*.jsonl).  The
U rows were taken with an experiment build that read the loads in flight per thread from
GEER_PROBE_U (4 / 8 / 16: the same rates); the library fixes 8."""
import os, json, sys
sys.path.insert(0, '.')
import paper_2312_06123_b200 as G
import torch
torch.cuda.init()
out = []
for U in ("4", "8", "16"):
    os.environ["GEER_PROBE_U"] = U
    for mb in (48, 128, 256, 512):
        for fl in (0, 1):
            r = G.er_probe_random_loads(mb << 20, fl, 32)
            out.append({"U": int(U), "mb": mb, "flavour": fl, "g_loads_per_s": r})
            print(json.dumps(out[-1]), flush=True)
