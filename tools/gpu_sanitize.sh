#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck / initcheck over every kernel family
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool"
  for part in stream small bucket multi grid@1 grid@2 grid@4 fill; do
    timeout 300 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $part 2>&1 | \
      grep -E "ok|ERROR SUMMARY|RACECHECK SUMMARY|Error|error|hazard" | head -20
  done
done > gpurun_out/r02_sanitize.txt 2>&1
echo done
