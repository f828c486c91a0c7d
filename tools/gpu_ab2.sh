#!/bin/bash
# A/B of a K1g change: parity subset, C5 stage at 8/64 clouds (grid@2, grid@4), traces
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-ab}.txt
{
timeout 1200 python -m pytest tests -m gpu -q -x -k "grid or mixed or adversarial or auto or suite or lidar or scale or fullscale" 2>&1 | tail -3
timeout 900 python tools/sweep_strong.py --n 50000 --iters 12500 --batches 8 64 --scheds grid@2 grid@4 2>&1
for s in grid@2; do
  for pr in f64 f32; do
    echo "-- $s $pr B=64"
    timeout 600 python tools/trace_multi.py --batch 64 --sched $s --precision $pr 2>&1 | tail -22
  done
done
} > $OUT 2>&1
echo done
