#!/bin/bash
# One GPU pass: parity tests, bench (JSON line), ncu launch list of one bench step,
# ncu --set full of the top kernels.  Everything lands in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref.json
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'attn_(fwd|bwd)' -s 6 -c 3 \
  -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'assign_kernel|pool_fwd|pool_bwd_kernel|nbr_kernel|radix_downsweep' -s 10 -c 8 \
  -o gpurun_out/prof_merge -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph > gpurun_out/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
fi
