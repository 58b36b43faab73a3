"""Writes profiles/traffic.json: DRAM bytes (read + write, ncu --set full) per C-ABI call of
the attention forward / backward, summed over the kernels of that call, keyed by the bench
workload.  usage: traffic_from_ncu.py prof_attn.ncu-rep <cfg_key> [source-note]"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else rep
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
ki, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = {"attn_fwd": 0.0, "attn_bwd": 0.0}
per = {}
for r in rows[2:]:
    name = r[ki]
    b = float(r[rd]) * scale[units[rd]] + float(r[wr]) * scale[units[wr]]
    op = "attn_fwd" if "attn_fwd" in name else "attn_bwd"
    tot[op] += b
    per[name[:60]] = b
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d[key] = {"attn_fwd": tot["attn_fwd"], "attn_bwd": tot["attn_bwd"], "kernels": per, "source": note,
          "note": "bytes per C-ABI call; the backward's small plan/finalize kernels are not included"}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[key], indent=1))
