mkdir -p gpurun_out
FFPS_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --batch 16 --no-exhaustive --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo torchrun=$?
cut -c1-600 gpurun_out/bench_2rank.json; tail -3 gpurun_out/bench_2rank.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_ref_2rank.json 2>&1; echo ref2=$?; cut -c1-300 gpurun_out/bench_ref_2rank.json
for NT in 512 1024; do
FFPS_BUCKET_NT=$NT FFPS_ALGO=bucket timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --reps 5 2>&1 | tail -1
done
