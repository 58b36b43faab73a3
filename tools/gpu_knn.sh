#!/bin/bash
# knn / merge-plan iteration: bit-exact parity tests + probe timings (+ fp64 rate)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-knn}
[ -x tools/micro/fp64_rate ] && ./tools/micro/fp64_rate
timeout 900 python -m pytest tests/test_index_gpu.py tests/test_merge_gpu.py tests/test_sweep_gpu.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 300 python tools/decoder_probe.py --batch 16 2>&1 | grep knn
timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --interp-images 0 --pretrain-batch 0 --tiny-batch 0 --e2e-steps 0 2>/dev/null | tail -1 | python -c "
import json,sys;d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phase_ms'], d['parity']['pass'])"
[ -n "$MODEL" ] && { timeout 1200 python -m pytest tests/test_model_gpu.py -m gpu -q -x > gpurun_out/${T}_model.log 2>&1; echo "model rc=$?"; tail -2 gpurun_out/${T}_model.log;
  timeout 300 python tools/pretrain_probe.py --batch 32 --steps 10 2>&1 | tail -2; }
exit 0
