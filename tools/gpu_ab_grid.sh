# A/B of K1g variants: parity (grid), C5 flash timings (uniform + lidar), trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid" 2>&1 | tail -1
for cloud in uniform lidar; do
  timeout 600 python tools/bench_configs.py $cloud --scheds grid --configs C5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['cloud'], d['config'], 'exh', round(d['exhaustive_ms'],2), 'flash', round(d['flash_p0.75_ms'],2))"
done
timeout 300 python tools/trace_multi.py --sched grid@2 2>&1 | tail -7
