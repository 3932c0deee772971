"""Summarise one kernel launch of an `ncu --set full` capture into the JSON that bench.py reads for
its roofline (profiles/ncu_<kind>_<config>_r02.json).

    python scripts/ncu_summary.py walks  <report.ncu-rep> <config> <walk_steps_json> [batch] > out.json
    python scripts/ncu_summary.py spmm   <report.ncu-rep> <config> <q>                      > out.json

walks: per-walk-step DRAM bytes and L2 / L1->L2 sectors of the captured K6 launch (batch `batch`
of a step, default 0), the step count of that launch taken from scripts/walk_batch_steps.py's
output for the same config (the library's own per-query stats: sum of 2 eta0 2^b ell_f).
spmm: DRAM bytes of the captured K9 launch and its achieved DRAM GB/s.
"""
import csv
import io
import json
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors.sum", "lts__t_sectors_srcunit_tex.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sectors_srcunit_ltcfabric.sum",
        "l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "launch__occupancy_limit_registers", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
        "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "sector": 1, "inst": 1, "%": 1, "": 1}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    return h, units, data


def value(h, units, r, k):
    i = h.index(k)
    v = float(r[i].replace(",", ""))
    return v * UNIT.get(units[i], 1)


def main():
    kind, report, config = sys.argv[1], sys.argv[2], sys.argv[3]
    h, units, data = raw(report)
    r = data[0]
    metrics = {k: f"{r[h.index(k)]} {units[h.index(k)]}".strip() for k in KEEP if k in h}
    t = value(h, units, r, "gpu__time_duration.sum")
    dram = value(h, units, r, "dram__bytes_read.sum") + value(h, units, r, "dram__bytes_write.sum")
    out = {"kernel": r[h.index("Kernel Name")].split("(")[0], "config": config, "report": report.split("/")[-1],
           "metrics": metrics, "duration_s": t, "dram_bytes": dram, "dram_gbs": dram / t / 1e9}
    if kind == "walks":
        steps_info = json.load(open(sys.argv[4]))
        b = int(sys.argv[5]) if len(sys.argv) > 5 else 0
        steps = steps_info[f"batch{b}_steps"]
        out.update({"batch": b, "walk_steps_in_launch": steps,
                    "walk_steps_source": "scripts/walk_batch_steps.py: sum over queries of 2 eta0 2^b ell_f",
                    "dram_bytes_per_walk_step": dram / steps,
                    "l2_sectors_per_walk_step": value(h, units, r, "lts__t_sectors.sum") / steps,
                    "walk_steps_per_s_under_ncu": steps / t})
        k = "l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum"
        if k in h:
            out["l1_to_l2_sectors_per_walk_step"] = value(h, units, r, k) / steps
    else:
        out["q"] = int(sys.argv[4])
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
