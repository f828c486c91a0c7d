#!/bin/bash
# ncu --set full of K0 (both kernels) + K1g on the C5 FlashFPS stage (binary64 on float coordinates)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
C="python tools/run_c5_stage.py f64"
timeout 600 $C > gpurun_out/r02_c5stage.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"fps_grid|bucket_kd" -s 2 -c 3 -o gpurun_out/r02_prof_c5 $C > gpurun_out/r02_ncu_full.log 2>&1; echo ncu=$?
