#!/bin/bash
# K1g phase traces: C5 flash stage and the minimal-table floor, binary32 and binary64-on-float
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for prec in f32 f64; do
  echo "== C5 $prec grid@2" ; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec
  echo "== floor $prec grid@2 (2048 points, 1024 iters)"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec --n 2048 --iters 1024
done > gpurun_out/r02b_trace.txt 2>&1
echo done
