cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export AFFMAE_GEMM_PAIR=1
timeout 60 python tools/gemm_dbg.py 512 256 128 2>&1 | tail -2
timeout 60 python tools/gemm_dbg.py 1000 384 264 2>&1 | tail -2
timeout 300 python -m pytest tests/test_linear_gpu.py -x -q 2>&1 | tail -15
timeout 300 python tools/gemm_probe.py 2>&1 | cut -c1-150
