#!/bin/bash
# Round-end evidence on one B200: smoke, every -m gpu test, the headline bench
# (+ LiDAR, reference arm, per-rank batches of the strong-scaling run), the
# multi-rank bench path, and every BASELINE config in binary64.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1; echo "smoke=$?" >> gpurun_out/${T}_smoke.txt
timeout 3000 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest=$?" >> gpurun_out/${T}_pytest.txt
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench=$?" >> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.json 2>&1
timeout 900 python bench.py --cloud lidar --no-cpu-baseline > gpurun_out/${T}_bench_lidar.json 2> gpurun_out/${T}_bench_lidar.err
for gb in 32 16 8; do
  timeout 600 python bench.py --global-batch $gb --no-exhaustive --no-cpu-baseline --no-extras > gpurun_out/${T}_bench_gb$gb.json 2>&1
done
FFPS_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-extras --exh-steps 1 > gpurun_out/${T}_dist2.json 2> gpurun_out/${T}_dist2.err; echo "dist2=$?" >> gpurun_out/${T}_dist2.err
timeout 2400 python tools/bench_configs.py uniform lidar > gpurun_out/${T}_configs.jsonl 2> gpurun_out/${T}_configs.err
timeout 600 python bench.py --n 24000 --dtype f32 --global-batch 16 --no-exhaustive --no-extras --no-cpu-baseline > gpurun_out/${T}_bench_c2_f32.json 2>&1
echo done
