timeout 1200 python -m pytest tests/test_model_gpu.py -q -m gpu --durations=10 > gpurun_out/r2c_model.log 2>&1
tail -80 gpurun_out/r2c_model.log
