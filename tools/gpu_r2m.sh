timeout 1200 python -m pytest tests/test_model_gpu.py tests/test_attention_gpu.py tests/test_linear_gpu.py tests/test_multi_rank_gpu.py -q -m gpu > gpurun_out/r2m_tests.log 2>&1
tail -5 gpurun_out/r2m_tests.log
python tools/pretrain_probe.py --batch 32 --steps 5 2>&1 | tail -2
