#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_workload.py
# (every kernel family); logs in gpurun_out/san/.
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all python scripts/sanitize_workload.py \
    > gpurun_out/san/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san/$tool.log | tail -1)"
done
