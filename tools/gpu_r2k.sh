for tool in memcheck racecheck synccheck initcheck; do
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/r2k_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "SUMMARY|ok$" gpurun_out/r2k_sanitize_$tool.log | tr '\n' ' '; echo
done
