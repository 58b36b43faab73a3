timeout 900 python -m pytest tests/test_affmae_module_gpu.py tests/test_integration_gpu.py tests/test_decoder_gpu.py tests/test_model_gpu.py -q -m gpu > gpurun_out/r2i_tests.log 2>&1
tail -30 gpurun_out/r2i_tests.log
