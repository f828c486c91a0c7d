#!/bin/bash
# AUTO schedule for binary64-on-float: every schedule over batch x n (iters = n/4)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python tools/sweep_auto.py --precision f32 --batches 1 8 16 32 64 --ns 2048 3072 4096 6000 8192 12000 16384 24000 --scheds small stream bucket grid@1 grid@2 auto > gpurun_out/auto32.jsonl 2>&1
timeout 1200 python tools/sweep_auto.py --precision f64 --batches 1 16 64 --ns 3072 5000 7000 --scheds small stream bucket grid@1 auto > gpurun_out/auto64b.jsonl 2>&1
echo done
