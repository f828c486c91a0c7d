mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --cloud lidar --no-cpu-baseline > gpurun_out/bench_lidar.json 2> gpurun_out/bench_lidar.err; echo benchl=$?
cat gpurun_out/bench_lidar.json; tail -3 gpurun_out/bench_lidar.err
