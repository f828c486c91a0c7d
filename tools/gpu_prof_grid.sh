# ncu source-level profile of K1g on the C5 flash stage (B=64, n=50000, 12500 iterations)
mkdir -p gpurun_out
C1="python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --reps 1"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k grid 2>&1 | tail -1
FFPS_ALGO=grid $C1 > gpurun_out/c1g.log 2>&1 && tail -1 gpurun_out/c1g.log && FFPS_ALGO=grid timeout 900 ncu --set full --clock-control none --import-source on -k regex:fps_grid -s 1 -c 1 -o gpurun_out/prof_k1g $C1 > gpurun_out/ncu_k1g.log 2>&1; echo ncu=$?
timeout 300 python tools/trace_multi.py --sched grid@2
