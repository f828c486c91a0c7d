#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -k "grid or mixed or adversarial or auto" 2>&1 | tail -3
for shape in "50000 12500" "75000 18750"; do
  set -- $shape
  timeout 900 python tools/sweep_strong.py --n $1 --iters $2 --batches 8 32 --scheds grid@2 grid@4 2>&1
done
timeout 600 python tools/trace_multi.py --batch 16 --sched grid@4 --precision f64 2>&1 | tail -30
} > gpurun_out/cl4c.txt 2>&1
echo done
