#!/bin/bash
# TMA staging of flagged buckets: parity + A/B (FFPS_GRID_STAGE=0 = off)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-stage}
{
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py -x -q -k "grid or mixed or hierarchy or kd" 2>&1 | tail -2
for st in 0 default; do
  if [ $st = default ]; then unset FFPS_GRID_STAGE; else export FFPS_GRID_STAGE=$st; fi
  echo "=== FFPS_GRID_STAGE=$st"
  timeout 300 python tools/sweep_strong.py --batches 64 --scheds grid@2 2>&1
  for prec in f32 f64; do echo "-- $prec"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec | grep -A6 "rounds \[9"; done
done
unset FFPS_GRID_STAGE
CS=/usr/local/cuda/bin/compute-sanitizer
echo "=== sanitizer smoke"
timeout 300 $CS --tool memcheck python tools/sanitize_run.py grid@2 2>&1 | tail -15
} > gpurun_out/${TAG}.txt 2>&1
echo done
