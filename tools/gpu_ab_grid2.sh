# K1g knobs: default / no prefetch / KM=16, C5 flash (uniform, lidar) + parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid" 2>&1 | tail -1
FFPS_GRID_KM=8 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid" 2>&1 | tail -1
run() {
  for cloud in uniform lidar; do
    timeout 600 python tools/bench_configs.py $cloud --scheds grid --configs C5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$1', d['cloud'], 'exh', round(d['exhaustive_ms'],2), 'flash', round(d['flash_p0.75_ms'],2))"
  done
}
run default

FFPS_GRID_KM=8 run km8
timeout 300 python tools/trace_multi.py --sched grid@2 2>&1 | tail -7
FFPS_GRID_KM=8 timeout 300 python tools/trace_multi.py --sched grid@2 2>&1 | tail -7
