#!/bin/bash
# parity subset + C5 stage sweep + one headline bench run
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-quick}.txt
{
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/sweep_strong.py --n 50000 --iters 12500 --batches 8 16 32 64 --scheds grid grid@2 grid@4 --precisions f64 f32 2>&1
timeout 900 python bench.py --no-cpu-baseline 2>&1 | tail -1
} > $OUT 2>&1
echo done
