#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=r02f
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest=$?" >> gpurun_out/${T}_pytest.txt
timeout 1200 python tools/sweep_auto.py --precision f64 --batches 1 16 64 --ns 4096 5000 6000 8192 12000 16384 --scheds small stream grid@1 auto > gpurun_out/${T}_auto64.jsonl 2>&1
timeout 2400 python tools/bench_configs.py uniform lidar --scheds auto > gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_configs.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo done
