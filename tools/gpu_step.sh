#!/bin/bash
# training-step iteration: model parity tests, AFFMAE-B probe (B=32), and an ncu launch list of
# the kernels matching $KREGEX (default: the row kernels) over one eager B=16 step
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-step}
[ -z "$SKIP_TEST" ] && { timeout 1500 python -m pytest tests/test_model_gpu.py tests/test_linear_gpu.py -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log; }
timeout 600 python tools/pretrain_probe.py --batch 32 --steps 10 > gpurun_out/${T}_pre.log 2>&1; echo "probe rc=$?"; tail -3 gpurun_out/${T}_pre.log
K=${KREGEX:-regex:ln_bwd|ln_fwd|gelu|colsum|splitk}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv --log-file gpurun_out/${T}_launches.csv \
  python tools/pretrain_probe.py --batch 16 --steps 1 --warmup 0 --no-graph > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
exit 0
