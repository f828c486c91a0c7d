#!/bin/bash
# A/B of library variants: K1g phase trace (C5 flash stage, f32 + f64) and timing per variant
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-ab}; shift
for v in default "$@"; do
  if [ "$v" = default ]; then unset FFPS_LIB_VARIANT; else export FFPS_LIB_VARIANT=$v; fi
  echo "=== variant $v"
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py -x -q -k "grid" 2>&1 | tail -1
  timeout 300 python tools/sweep_strong.py --batches 64 --scheds grid@2 2>&1
  for prec in f32 f64; do echo "-- $prec"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec | grep -A6 "rounds \[9"; done
done > gpurun_out/${TAG}.txt 2>&1
echo done
