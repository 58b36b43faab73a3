#!/bin/bash
# compute-sanitizer over every kernel family (small shapes): memcheck / racecheck / synccheck / initcheck
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-san}
for tool in memcheck racecheck synccheck initcheck; do
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_probe.py > gpurun_out/${T}_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "SUMMARY|ok$" gpurun_out/${T}_$tool.log | tr '\n' ' '; echo
done
