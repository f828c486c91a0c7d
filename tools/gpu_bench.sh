mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref=$?
cat gpurun_out/bench_ref.json
B2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --exh-steps 1"
timeout 600 $B2 > gpurun_out/b2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B2 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fps_bucket -c 1 -o gpurun_out/prof_bench_k1b $B2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
