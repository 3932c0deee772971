"""DRAM bytes of the SMM head's kernels (push, y-table build and head bookkeeping) in one full
er_query_batch call, from an ncu launch list with dram__bytes_read/write per launch
(scripts/gpu_head_dram.sh): the launches between the first and the second K1 (k_setup) are the
first call of bench.py (its timed step).  -> profiles/ncu_smm_head_<config>_r02.json

    python scripts/head_dram.py <launches.csv> <config>
"""
import collections
import csv
import json
import re
import sys

HEAD = re.compile(r"k_bkt_|k_y|k_first_wave|k_compact|k_seg_max2|k_seg_off|k_seglen|k_ent_deg|k_decide|"
                  r"k_scan_|k_query_pairs|k_setup|k_flag_phase|k_init_frontier|k_dense_")
path, config = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
setups = [int(r[ii]) for r in rows[1:] if "k_setup" in r[ki] and r[mi] == "gpu__time_duration.sum"]
lo, hi = setups[0], setups[1]
agg = collections.defaultdict(lambda: {"read": 0.0, "write": 0.0, "ms": 0.0, "launches": 0})
for r in rows[1:]:
    if not (lo <= int(r[ii]) < hi) or not HEAD.search(r[ki]):
        continue
    name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
    v = float(r[vi].replace(",", ""))
    if r[mi] == "dram__bytes_read.sum":
        agg[name]["read"] += v
    elif r[mi] == "dram__bytes_write.sum":
        agg[name]["write"] += v
    elif r[mi] == "gpu__time_duration.sum":   # ns
        agg[name]["ms"] += v * 1e-6
        agg[name]["launches"] += 1
tot_b = sum(a["read"] + a["write"] for a in agg.values())
tot_ms = sum(a["ms"] for a in agg.values())
out = {"config": config, "source": f"{path} (launch IDs {lo}..{hi - 1}: the first full call)",
       "dram_bytes_per_call": tot_b, "kernel_ms_per_call": tot_ms,
       "dram_gbs_over_kernel_time": tot_b / tot_ms / 1e6,
       "by_kernel": {k: {"dram_gb": round((a["read"] + a["write"]) / 1e9, 3), "ms": round(a["ms"], 3),
                         "launches": a["launches"]}
                     for k, a in sorted(agg.items(), key=lambda x: -(x[1]["read"] + x[1]["write"]))}}
print(json.dumps(out, indent=1))
