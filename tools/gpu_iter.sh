#!/bin/bash
# iteration loop: parity of every GPU schedule suite that the kernels touch,
# C5 greedy timings (64 and 16 clouds) and an ncu launch list of one C5 stage
mkdir -p gpurun_out
T=${1:-k0}
{
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_coverage.py -q -x 2>&1 | tail -1
timeout 300 python tools/sweep_strong.py --batches 64 16 --scheds grid@2 2>&1
} > gpurun_out/${T}.txt 2>&1
timeout 300 python tools/run_c5_stage.py f64 > gpurun_out/${T}_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/run_c5_stage.py f64 > gpurun_out/${T}_ncu.log 2>&1
echo done
