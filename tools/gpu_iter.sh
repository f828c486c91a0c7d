#!/bin/bash
# iteration loop: parity of every GPU suite the kernels touch, C5 greedy timings
# (64 and 16 clouds), K1g phase traces, and an ncu launch list of one C5 stage
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-iter}
{
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_coverage.py tests/test_gpu_fullscale.py -q -x 2>&1 | tail -1
timeout 300 python tools/sweep_strong.py --batches 64 16 --scheds grid@2 2>&1
for prec in f32 f64; do echo "-- $prec"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec | grep -A6 "rounds \[9"; done
} > gpurun_out/${T}.txt 2>&1
timeout 300 python tools/run_c5_stage.py f64 > gpurun_out/${T}_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/run_c5_stage.py f64 > gpurun_out/${T}_ncu.log 2>&1
echo done
