# K1g iteration: grid parity, phase trace, C5 timings (uniform + LiDAR)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "grid" 2>&1 | tail -2
timeout 300 python tools/trace_multi.py --sched grid@2 2>&1 | tail -7
for cloud in uniform lidar; do
  timeout 600 python tools/bench_configs.py $cloud --scheds grid --configs ${CONFIGS:-C5} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:3], d['cloud'], 'exh', round(d['exhaustive_ms'],2), 'flash', round(d['flash_p0.75_ms'],2))"
done
if [ -n "$KM_AB" ]; then
  for km in $KM_AB; do
    FFPS_GRID_KM=$km timeout 600 python tools/bench_configs.py uniform --scheds grid --configs C5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('km$km', d['config'][:3], d['cloud'], 'exh', round(d['exhaustive_ms'],2), 'flash', round(d['flash_p0.75_ms'],2))"
  done
fi
