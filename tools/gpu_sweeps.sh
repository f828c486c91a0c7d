#!/bin/bash
# Sweeps behind the AUTO rule, the strong-scaling shapes and the divergence report
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python tools/sweep_auto.py --precision f64 --batches 1 8 16 32 64 --ns 1024 2048 4096 6000 8192 12000 16384 24000 --scheds small stream bucket grid@1 grid@2 auto > gpurun_out/sweep_auto_f64.jsonl 2>&1
timeout 2400 python tools/sweep_auto.py --precision f32 --batches 1 8 16 32 64 --ns 2048 3072 4096 6000 8192 12000 16384 24000 --scheds small stream bucket grid@1 grid@2 auto > gpurun_out/sweep_auto_f32.jsonl 2>&1
timeout 900 python tools/sweep_strong.py > gpurun_out/sweep_strong.jsonl 2>&1
timeout 900 python tools/divergence.py > gpurun_out/divergence.jsonl 2>&1
echo done
