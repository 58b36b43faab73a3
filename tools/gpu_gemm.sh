cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_linear_gpu.py -x -q > gpurun_out/pytest_linear.log 2>&1; echo "linear tests rc=$?"
tail -30 gpurun_out/pytest_linear.log
timeout 300 python tools/gemm_probe.py > gpurun_out/gemm_tc.jsonl 2>&1; echo "probe rc=$?"
cat gpurun_out/gemm_tc.jsonl
