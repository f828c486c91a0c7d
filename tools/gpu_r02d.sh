#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fullscale.py -q -k lidar > gpurun_out/r02d_lidar.txt 2>&1; echo "rc=$?" >> gpurun_out/r02d_lidar.txt
timeout 900 python tools/divergence.py > gpurun_out/r02_divergence.jsonl 2> gpurun_out/r02_divergence.err
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
bash tools/gpu_sanitize.sh
echo done
