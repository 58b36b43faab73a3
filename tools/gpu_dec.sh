#!/bin/bash
# decoder attention iteration: gattn parity tests + decoder probe timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-dec}
[ -z "$SKIP_TEST" ] && { timeout 900 python -m pytest tests/test_gattn_gpu.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log; }
timeout 300 python tools/decoder_probe.py --batch 16 > gpurun_out/${T}_probe.log 2>&1; echo "probe rc=$?"; cat gpurun_out/${T}_probe.log | tail -12
[ -n "$MODEL" ] && { timeout 1200 python -m pytest tests/test_model_gpu.py -m gpu -q -x > gpurun_out/${T}_model.log 2>&1; echo "model rc=$?"; tail -3 gpurun_out/${T}_model.log;
  timeout 300 python tools/pretrain_probe.py --batch 32 --steps 10 > gpurun_out/${T}_pre.log 2>&1; tail -3 gpurun_out/${T}_pre.log; }
exit 0
