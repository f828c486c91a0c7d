# K1g with the two-level bucket-group index: parity, C5 timings, traces
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cloud in uniform lidar; do
  timeout 600 python tools/bench_configs.py $cloud --scheds grid bucket --configs C3 C4 C5 2>/dev/null | cut -c1-330
done
timeout 300 python tools/trace_multi.py --sched grid@2 --cloud lidar
timeout 300 python tools/trace_multi.py --sched grid@2
