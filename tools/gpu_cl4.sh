#!/bin/bash
# 4 CTAs per cloud with KM = 16: parity + per-cloud time at the strong-scaling batches
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_adversarial.py -q -x -k "grid" 2>&1 | tail -1
timeout 900 python tools/sweep_strong.py --batches 8 16 32 37 64 --scheds grid@2 grid@4 grid@4/km8 2>&1
for prec in f32 f64; do echo "-- $prec grid@4 B=16"; timeout 120 python tools/trace_multi.py --sched grid@4 --batch 16 --precision $prec | grep -A6 "rounds \[9"; done
} > gpurun_out/cl4.txt 2>&1
echo done
