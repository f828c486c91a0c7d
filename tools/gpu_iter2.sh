#!/bin/bash
# iteration loop: K1g parity (all grid schedules, f32/f64/mixed) + C5 greedy timing + phase trace
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-iter}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py -x -q -k "grid or Grid or mixed or hierarchy or kd" > gpurun_out/${TAG}_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.txt
timeout 300 python tools/sweep_strong.py --batches 64 8 --scheds grid@2 grid@1 > gpurun_out/${TAG}_strong.jsonl 2>&1
for prec in f32 f64; do echo "== C5 $prec grid@2"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec; done > gpurun_out/${TAG}_trace.txt 2>&1
echo done
