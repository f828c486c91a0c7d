#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
for shape in "25000 6250" "37500 9375" "75000 18750" "100000 25000"; do
  set -- $shape
  timeout 900 python tools/sweep_strong.py --n $1 --iters $2 --batches 4 8 16 32 --scheds grid@2 grid@4 2>&1
done
} > gpurun_out/cl4b.txt 2>&1
echo done
