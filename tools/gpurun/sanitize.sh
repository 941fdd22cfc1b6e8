#!/bin/bash
# compute-sanitizer racecheck / memcheck / synccheck over tools/sanitize_run.py (every tile width,
# both goal modes, oracle alongside, comparison schemes, chunked runs, goal changes)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
