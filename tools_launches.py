"""Per-kernel time of ONE step from an ncu launch list (--metrics gpu__time_duration.sum --csv).
Usage: python tools_launches.py launches.csv [top] [step_index]
The step is the span from the step_index-th k_setup launch (0-based; default 3 = the first timed
step of `bench.py --warmup 3`) to the next k_setup."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
R = rows[hi + 1:]
ki = h.index('Kernel Name')
mi = h.index('Metric Value')
seq = [(r[ki], float(r[mi].replace(',', ''))) for r in R if len(r) > mi]
idxs = [i for i, (n, v) in enumerate(seq) if 'k_setup' in n]
si = int(sys.argv[3]) if len(sys.argv) > 3 else 3
b0, b1 = idxs[si], idxs[si + 1]
agg = collections.defaultdict(float)
c = collections.Counter()
for n, v in seq[b0:b1]:
    n = n.split('(')[0][:90]
    agg[n] += v
    c[n] += 1
T = sum(agg.values())
for n, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{v/1e3:9.1f} us {100*v/T:5.1f}% x{c[n]:3d} {n}")
print('total us', T / 1e3, 'launches', b1 - b0)
