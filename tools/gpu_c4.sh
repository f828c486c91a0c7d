#!/bin/bash
# BASELINE configs[3]: C4 (N=300K, budgets 75000/18750/4687/1171), global batch 32 on
# one GPU and the 4-cloud per-rank shape of the 8-GPU run; uniform and LiDAR
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for cloud in uniform lidar; do
  for gb in 32 4; do
    timeout 900 python bench.py --n 300000 --global-batch $gb --cloud $cloud --no-cpu-baseline --no-extras \
      $( [ $gb = 4 ] && echo --no-exhaustive ) > gpurun_out/c4_${cloud}_gb$gb.json 2>&1
  done
done
echo done
