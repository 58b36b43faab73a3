"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: launch_summary.py launches.csv [n_steps_to_skip_fraction]
Prints per-kernel count / total / share over our kernels (torch RNG/copy kernels dropped)."""
import collections
import csv
import io
import sys

path = sys.argv[1]
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:])))
        if r["Metric Name"] == "gpu__time_duration.sum"]
skip = ("at::", "native::", "cutlass", "gemm", "elementwise", "Memcpy", "memcpy")
ours = [r for r in rows if not any(s in r["Kernel Name"] for s in skip)]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
ours = ours[int(len(ours) * frac):]
unit = rows[0]["Metric Unit"]
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
agg = collections.OrderedDict()
for r in ours:
    n = r["Kernel Name"].split("(")[0]
    n = n.replace("void ", "").replace("affmae_b200::", "")[:70]
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
print(f"{len(rows)} launches total, {len(ours)} of ours, {tot:.1f} us")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:72s} {c:5d} {t:10.1f} us {100 * t / tot:5.1f}%")
