timeout 900 python -m pytest tests/test_model_gpu.py tests/test_multi_rank_gpu.py -q -m gpu -x > gpurun_out/r2l_tests.log 2>&1
tail -3 gpurun_out/r2l_tests.log
python tools/pretrain_probe.py --batch 32 --steps 5 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_pretrain_launches.csv python tools/pretrain_probe.py --batch 16 --steps 1 --warmup 0 --no-graph > /dev/null 2>&1
