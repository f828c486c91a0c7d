# kd-tree K0: parity (all schedules + coverage), then kd vs Morton timings and traces
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for build in kd morton; do
  if [ $build = morton ]; then export FFPS_BUCKET_BUILD=morton; else unset FFPS_BUCKET_BUILD; fi
  for cloud in uniform lidar; do
    for s in grid bucket; do
      r=$(timeout 600 python tools/bench_configs.py $cloud --scheds $s --configs C5 2>/dev/null | tail -1 | cut -c1-330)
      echo "$build $cloud $s: $r"
    done
  done
done
unset FFPS_BUCKET_BUILD
timeout 300 python tools/trace_multi.py --sched grid@2 --cloud lidar
timeout 300 python tools/trace_multi.py --sched grid@2
