#!/bin/bash
# ncu launch list of a short headline bench run (one ncu per gpurun call)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-exhaustive --no-extras"
timeout 900 $B2 > gpurun_out/r02_b2.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B2 > gpurun_out/r02_ncu_launch.log 2>&1; echo ncu=$?
