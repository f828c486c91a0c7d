# A/B of library variants (tools/build_variant.sh): grid parity + trace + C5 timings each
mkdir -p gpurun_out
for v in default $VARIANTS; do
  if [ "$v" = default ]; then unset FFPS_LIB_VARIANT; else export FFPS_LIB_VARIANT=$v; fi
  echo "== $v"
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid" 2>&1 | tail -1
  timeout 300 python tools/trace_multi.py --sched grid@2 2>&1 | tail -6 | head -2
  for cloud in uniform lidar; do
    timeout 600 python tools/bench_configs.py $cloud --scheds grid --configs ${CONFIGS:-C5} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'][:3], d['cloud'], 'exh', round(d['exhaustive_ms'],2), 'flash', round(d['flash_p0.75_ms'],2))"
  done
done
