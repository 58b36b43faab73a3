timeout 1800 python -m pytest tests/test_sweep_gpu.py tests/test_integration_gpu.py tests/test_io_gpu.py tests/test_index_gpu.py tests/test_merge_gpu.py -q -m gpu --durations=20 > gpurun_out/r2b_sweep.log 2>&1
tail -40 gpurun_out/r2b_sweep.log
