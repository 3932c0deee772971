"""Per-kernel totals of the last query batch in an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    with open(f) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = [(r["Kernel Name"][:70], float(r["Metric Value"])) for r in csv.DictReader(lines)
            if r["Metric Name"] == "gpu__time_duration.sum"]
    starts = [i for i, (n, _) in enumerate(rows) if "k_setup" in n]
    last = rows[starts[-1]:] if starts else rows
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in last:
        agg[n][0] += 1
        agg[n][1] += v
    print(f, "total us %.1f" % (sum(v for _, v in last) / 1e3))
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
        print(f"  {v / 1e3:9.1f} us  x{c:3d}  {n}")
