#!/bin/bash
# Launch-list timing of the attention kernels under experiment flags.
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for f in ${FLAGS:-0 1}; do
  AFFMAE_EXP=$f timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/exp_$f.csv \
    python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph > /dev/null 2>&1
  echo "== AFFMAE_EXP=$f"; python tools/launch_summary.py gpurun_out/exp_$f.csv | grep attn_
done
