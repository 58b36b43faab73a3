#!/bin/bash
# Quick GPU pass: attention parity tests first (short timeout: a pipeline deadlock must not
# burn the box), then the full GPU suite, the bench line and a launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
timeout 300 python -m pytest tests/test_attention_gpu.py -x -q > gpurun_out/pytest_attn.log 2>&1; echo "attn tests rc=$?"
tail -5 gpurun_out/pytest_attn.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/pytest_gpu.log
fi
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph --interp-images 0 > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
fi
if [ -n "$NCU_FULL" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-3} \
  -o gpurun_out/prof_full -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph --interp-images 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
