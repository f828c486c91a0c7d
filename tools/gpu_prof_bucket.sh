mkdir -p gpurun_out
C1="python tools/sweep.py --batch 64 --n 50000 --cloud-n 50000 --iters 3000 --reps 1"
FFPS_ALGO=bucket $C1 > gpurun_out/c1b.log 2>&1 && FFPS_ALGO=bucket ncu --set full --clock-control none --import-source on -k regex:fps_bucket -s 1 -c 1 -o gpurun_out/prof_k1b $C1 > gpurun_out/ncu_k1b.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_k1b.log
