#!/bin/bash
# KM = 8 vs 16 on the small K1g tables of C2 / C3 (binary64 on float)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
for shape in "6000 1500 16" "24000 6000 16" "25000 6250 8" "12500 3125 8" "8192 2048 16"; do
  set -- $shape
  timeout 300 python tools/sweep_strong.py --n $1 --iters $2 --batches $3 --scheds grid@1 grid@1/km8 grid@2 grid@2/km8 --precisions f64 2>&1
done
} > gpurun_out/small_km.txt 2>&1
echo done
