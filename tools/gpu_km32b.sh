#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
export FFPS_GRID_KM=32
for prec in f32 f64; do echo "-- KM32 $prec"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec | tail -8; done
} > gpurun_out/km32b.txt 2>&1
echo done
