#!/bin/bash
# K1g bucket size class x CTAs per cloud on LiDAR-like frames (binary64)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-ppl_lidar}.txt
{
for shape in "50000 12500 200000" "75000 18750 300000" "100000 25000 400000"; do
  set -- $shape
  for ppl in 1 2 4; do
    echo "=== PPL $ppl n $1"
    FFPS_GRID_PPL=$ppl timeout 1200 python tools/sweep_strong.py --cloud lidar --cloud-n $3 --n $1 --iters $2 --batches 16 64 --scheds grid@2 grid@4 --precisions f64 2>&1 | sed "s/^{/{\"ppl\": $ppl, /"
  done
done
} > $OUT 2>&1
echo done
