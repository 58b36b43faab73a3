"""Maps an ncu SASS source-page CSV onto CUDA source lines (nvdisasm -g line info).
usage: ncu_lines.py <ncu source csv> <cubin> <mangled kernel> [kernel-index]"""
import csv, os, re, subprocess, sys
from collections import Counter
csvf, cubin, kname = sys.argv[1:4]
kidx = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
st = [i for i, l in enumerate(sass) if l.startswith("//---") and ".text." + kname + " " in l + " "][0]
en = [i for i, l in enumerate(sass) if i > st + 5 and l.startswith("//-----")]
en = en[0] if en else len(sass)
a2l, cur = {}, None
for l in sass[st:en]:
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
hi = starts[kidx]
end = starts[kidx + 1] - 1 if kidx + 1 < len(starts) else len(rows)
hdr = rows[hi]
ia, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = None
ci, cs = Counter(), Counter()
# EXTRA="L1 Wavefronts Shared,L1 Wavefronts Shared Excessive": also sum these
# columns per line and rank by the first of them
extra = [c for c in os.environ.get("EXTRA", "").split(",") if c]
ix = [hdr.index(c) for c in extra]
ce = [Counter() for _ in extra]
for r in rows[hi + 1:end]:
    try:
        a = int(r[0], 16); n = float(r[ia] or 0); s = float(r[ist] or 0)
    except (ValueError, IndexError):
        continue
    base = a if base is None else base
    k = a2l.get(a - base, "?")
    ci[k] += n; cs[k] += s
    for c, j in zip(ce, ix):
        try:
            c[k] += float(r[j] or 0)
        except ValueError:
            pass
tot, ts = sum(ci.values()), sum(cs.values())
import os
srcdir = os.environ.get("SRCDIR") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2602_16249_b200", "csrc")
src = {}
for k in list(ci):
    f = k.split(":")[0]
    if f not in src and os.path.exists(os.path.join(srcdir, f)):
        src[f] = open(os.path.join(srcdir, f)).read().split("\n")
print(f"total warp-instructions {tot/1e6:.2f}M")
if extra:
    te = [sum(c.values()) or 1 for c in ce]
    print("extra totals:", ", ".join(f"{n}={t/1e6:.2f}M" for n, t in zip(extra, te)))
    for k, _ in sorted(ce[0].items(), key=lambda kv: -kv[1])[:int(os.environ.get("TOP", 30))]:
        f, l = (k.split(":") + ["0"])[:2]
        text = src[f][int(l) - 1].strip()[:60] if f in src else ""
        vals = " ".join(f"{100*c[k]/t:5.1f}%" for c, t in zip(ce, te))
        print(f"{vals} {k}: {text}")
    sys.exit(0)
for k, v in sorted(ci.items(), key=lambda kv: -(kv[1] / tot + cs[kv[0]] / ts))[:int(os.environ.get("TOP", 30))]:
    f, l = (k.split(":") + ["0"])[:2]
    text = src[f][int(l) - 1].strip()[:70] if f in src else ""
    print(f"{100*v/tot:5.1f}% inst {100*cs[k]/ts:5.1f}% stall {k}: {text}")
