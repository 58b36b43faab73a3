set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_sweep_gpu.py tests/test_integration_gpu.py -q -x -m gpu --durations=15 > gpurun_out/r2a_sweep.log 2>&1
tail -30 gpurun_out/r2a_sweep.log
for tool in memcheck racecheck synccheck initcheck; do
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/r2a_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -5 gpurun_out/r2a_sanitize_$tool.log
done
