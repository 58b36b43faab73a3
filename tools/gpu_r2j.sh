timeout 900 python -m pytest tests/test_multi_rank_gpu.py tests/test_model_gpu.py -q -m gpu -x > gpurun_out/r2j_tests.log 2>&1
tail -15 gpurun_out/r2j_tests.log
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
tail -3 gpurun_out/r2j_bench.err; echo "bench wall $(( $(date +%s) - T0 )) s"
