#!/bin/bash
# attention iteration: parity tests of the cluster attention + bench phase times (+ optional ncu of bwd)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-attn}
[ -z "$SKIP_TEST" ] && timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_sweep_gpu.py tests/test_integration_gpu.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${T}_pytest.log
B="python bench.py --steps 30 --warmup 3 --no-cpu-baseline --interp-images 0 --pretrain-batch 0 --tiny-batch 0 --e2e-steps 0"
timeout 600 $B > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['phase_ms'], d['roofline']['frac'], d.get('parity',{}).get('pass'))"
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'attn_(bwd_q|bwd_kv)_kernel' -s 3 -c 3 \
  -o gpurun_out/${T}_prof -f python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-graph --interp-images 0 --pretrain-batch 0 --tiny-batch 0 --no-parity > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
fi
