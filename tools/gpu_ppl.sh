#!/bin/bash
# K1g bucket size class (32 x PPL points) x CTAs per cloud x candidate count, binary64
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-ppl}.txt
PREC=${2:-f64}
{
for shape in "25000 6250" "37500 9375" "50000 12500" "75000 18750" "100000 25000" "150000 37500"; do
  set -- $shape
  for ppl in 1 2 4; do
    echo "=== PPL $ppl n $1"
    FFPS_GRID_PPL=$ppl timeout 900 python tools/sweep_strong.py --n $1 --iters $2 --batches 16 64 --scheds grid@1 grid@2 grid@4 --precisions $PREC 2>&1 | sed "s/^{/{\"ppl\": $ppl, /"
  done
done
} > $OUT 2>&1
echo done
