#!/bin/bash
# CTAs-per-cloud crossover of K1g (AUTO's grid_cluster threshold)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
for shape in "30000 7500" "37500 9375" "42000 10500" "46000 11500" "50000 12500"; do
  set -- $shape
  timeout 900 python tools/sweep_strong.py --n $1 --iters $2 --batches 8 32 --scheds grid@2 grid@4 2>&1
done
} > gpurun_out/${1:-cl4b}.txt 2>&1
echo done
