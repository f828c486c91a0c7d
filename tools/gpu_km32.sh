#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
export FFPS_GRID_KM=32
timeout 900 python -m pytest tests/test_gpu_mixed.py -q -x -k "grid_sizes" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bucketed_schedule_sizes or degenerate" 2>&1 | tail -3
for km in 16 32; do
  export FFPS_GRID_KM=$km; echo "=== KM=$km"
  timeout 300 python tools/sweep_strong.py --batches 64 8 --scheds grid@2 2>&1
  for prec in f32 f64; do echo "-- $prec"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec | grep -A7 "rounds \[9"; done
done
} > gpurun_out/km32.txt 2>&1
echo done
