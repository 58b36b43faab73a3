timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_sweep_gpu.py -q -m gpu -x -k "attn or attention" > gpurun_out/r2o_tests.log 2>&1
tail -3 gpurun_out/r2o_tests.log
python bench.py --pretrain-batch 0 --tiny-batch 0 --no-cpu-baseline --interp-images 0 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['phase_ms'], d['roofline']['frac'], d['parity']['pass'])"
