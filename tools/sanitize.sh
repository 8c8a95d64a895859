#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# tools/sanitize_run.py (every kernel family, small sizes). Run under gpurun;
# logs land in gpurun_out/sanitize_<tool>.log.
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/status.txt
done
