#!/bin/bash
# Training-step check: model + linear tests, then the AFFMAE-B 1024^2 step (64 images, graph)
# with the default GEMMs, then the launch list of one eager B=16 step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_linear_gpu.py tests/test_model_gpu.py tests/test_merge_tokens_gpu.py -x -q > gpurun_out/pytest_step.log 2>&1; echo "step tests rc=$?"
tail -4 gpurun_out/pytest_step.log
timeout 600 python tools/pretrain_probe.py --batch 64 --steps 5 > gpurun_out/pretrain_tc.log 2>&1; echo "probe rc=$?"; tail -3 gpurun_out/pretrain_tc.log
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pretrain_launches.csv \
  python tools/pretrain_probe.py --batch 16 --steps 1 --no-graph > gpurun_out/ncu_pretrain.log 2>&1; echo "ncu pretrain rc=$?"
fi
