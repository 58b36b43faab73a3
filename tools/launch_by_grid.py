"""Summarise an ncu --csv launch list per (kernel, grid): count, mean / min / max us.
    python tools/launch_by_grid.py gpurun_out/x_launches.csv [substring]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
d = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi and (len(sys.argv) < 3 or sys.argv[2] in r[ki]):
        d[(r[ki].split('(')[0][:70], r[gi])].append(float(r[vi].replace(',', '')) / 1e3)
tot = 0.0
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    tot += sum(v)
    print(f"{sum(v):9.1f} us {len(v):4d}x mean {sum(v) / len(v):7.1f} min {min(v):7.1f} max {max(v):7.1f}  {k[0]} {k[1]}")
print(f"total {tot:.1f} us")
