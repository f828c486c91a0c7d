# torchrun paths of bench.py on a 1-GPU box: 2 ranks sharing the GPU (gloo; exercises the
# barriers, max-over-ranks timing and the index gather; not a scaling number) and 1 rank
mkdir -p gpurun_out
FFPS_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --exh-steps 1 > gpurun_out/dist2.json 2> gpurun_out/dist2.err; echo dist=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --exh-steps 1 > gpurun_out/dist1.json 2> gpurun_out/dist1.err; echo dist1=$?
