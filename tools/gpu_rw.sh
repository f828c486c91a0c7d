#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
timeout 1200 python -m pytest tests -m gpu -q -x -k "grid or mixed or adversarial or suite or fullscale or lidar" 2>&1 | tail -1
bash tools/gpu_variants.sh rw_var rw8 rw16 > /dev/null 2>&1; cat gpurun_out/rw_var.txt
echo "-- trace default C5 grid@2 f64"; timeout 300 python tools/trace_multi.py --batch 64 --sched grid@2 --precision f64 2>&1 | sed -n '/^rounds \[9/,/^loop/p'
} > gpurun_out/rw.txt 2>&1
echo done
