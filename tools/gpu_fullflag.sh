#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/fullflag.txt
{
for v in default fullflag; do
  echo "=== variant $v"
  if [ "$v" = default ]; then unset FFPS_LIB_VARIANT; else export FFPS_LIB_VARIANT=$v; fi
  timeout 900 python tools/sweep_strong.py --n 50000 --iters 12500 --batches 16 64 --scheds grid@2 grid@4 --precisions f64 2>&1
  echo "-- trace C5 grid@2 B=64"; timeout 300 python tools/trace_multi.py --batch 64 --sched grid@2 --precision f64 2>&1 | grep -A5 "^rounds \[9"
  echo "-- trace C5 grid@4 B=16"; timeout 300 python tools/trace_multi.py --batch 16 --sched grid@4 --precision f64 2>&1 | grep -A5 "^rounds \[9"
  echo "-- trace C3 grid@2 B=8"; timeout 300 python tools/trace_multi.py --batch 8 --n 25000 --iters 6250 --cloud-n 100000 --sched grid@2 --precision f64 2>&1 | tail -14
done
} > $OUT 2>&1
echo done
