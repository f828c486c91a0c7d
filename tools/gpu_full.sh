mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref=$?
timeout 900 python bench.py --cloud lidar --no-cpu-baseline > gpurun_out/bench_lidar.json 2> gpurun_out/bench_lidar.err; echo benchl=$?
timeout 1500 python tools/bench_configs.py uniform lidar > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo cfg=$?
B2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --exh-steps 1"
timeout 600 $B2 > gpurun_out/b2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B2 > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fps_grid -c 1 -o gpurun_out/prof_bench_k1g $B2 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none -k regex:bucket_kd -c 2 -o gpurun_out/prof_bench_k0 python tools/run_grid.py --reps 1 > gpurun_out/ncu_k0.log 2>&1; echo ncu3=$?
timeout 300 python tools/trace_multi.py --sched grid@2 > gpurun_out/trace_grid.txt 2>&1; echo trace=$?
