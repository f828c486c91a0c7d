#!/bin/bash
# exact bucket size class A/B at the ambiguous table sizes, uniform and LiDAR, binary64
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-ppl2}.txt
{
for cloud in uniform lidar; do
  for shape in "50000 12500 200000" "75000 18750 300000"; do
    set -- $shape
    for ppl in 1 2 4; do
      echo "=== $cloud PPL $ppl n $1"
      FFPS_GRID_PPL=$ppl timeout 1200 python tools/sweep_strong.py --cloud $cloud --cloud-n $3 --n $1 --iters $2 --batches 16 64 --scheds grid@2 grid@4 --precisions f64 2>&1 | sed "s/^{/{\"cloud\": \"$cloud\", \"ppl\": $ppl, /"
    done
  done
done
} > $OUT 2>&1
echo done
