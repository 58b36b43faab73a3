#!/bin/bash
# dW side-stream overlap check: model tests, pretrain probe with / without the overlap
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_model_gpu.py tests/test_multi_rank_gpu.py tests/test_affmae_module_gpu.py -m gpu -q -x > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2f_pytest.log
for B in 32 64; do
  timeout 300 python tools/pretrain_probe.py --batch $B --steps 10 > gpurun_out/r2f_probe_$B.log 2>&1; echo "probe $B rc=$?"; tail -3 gpurun_out/r2f_probe_$B.log
  AFFMAE_NO_DW_OVERLAP=1 timeout 300 python tools/pretrain_probe.py --batch $B --steps 10 > gpurun_out/r2f_probe_${B}_noov.log 2>&1; echo "probe $B noov rc=$?"; tail -3 gpurun_out/r2f_probe_${B}_noov.log
done
