"""Key metrics of every kernel in an ncu --set full report (run here, no GPU needed).
usage: ncu_summary.py report.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]
ki = hdr.index("Kernel Name")
for r in rows[2:]:
    name = r[ki]
    if pat and not pat.search(name):
        continue
    print(f"--- {name[:110]}")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:64s} {r[i]:>16s} {units[i]}")
