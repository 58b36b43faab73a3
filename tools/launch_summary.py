"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time per kernel family."""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    gi = h.index("Grid Size")
    out = []
    for r in rows[hdr + 1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        out.append((r[ki], v / 1e3, r[gi]))  # us
    return out


def family(n):
    if "cutlass" in n:
        for k, lab in (("StreamK", "gemm(streamK)"),):
            pass
        tags = []
        if "LinearCombination<float" in n:
            tags.append("gemm bwd fp32-out")
        elif "LinearCombination<cutlass::bfloat16" in n:
            tags.append("gemm bwd dX bf16")
        elif "GELU" in n:
            tags.append("gemm fwd +bias+GELU")
        else:
            tags.append("gemm fwd")
        return tags[0]
    return re.sub(r"\(.*", "", re.sub(r"<.*?>", "", n)).replace("void ", "").strip()


if __name__ == "__main__":
    seq = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for n, t, g in seq:
        f = family(n)
        agg[f][0] += 1
        agg[f][1] += t
        tot += t
    print(f"{len(seq)} launches, {tot / 1e3:.2f} ms of kernel time")
    for f, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
        print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% {c:5d}  {f}")
