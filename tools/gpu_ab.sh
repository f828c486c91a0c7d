#!/bin/bash
# A/B of library variants (tools/build_variant.sh): parity of the default build,
# then per variant C5 timings (64 and 16 clouds) and K1g phase traces
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
TAG=${1:-ab}; shift
{
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_fullscale.py tests/test_gpu_adversarial.py -q -x 2>&1 | tail -1
for v in default "$@"; do
  if [ "$v" = default ]; then unset FFPS_LIB_VARIANT; else export FFPS_LIB_VARIANT=$v; fi
  echo "=== variant $v"
  timeout 300 python tools/sweep_strong.py --batches 64 16 --scheds grid@2 2>&1
  for prec in f32 f64; do echo "-- $prec"; timeout 120 python tools/trace_multi.py --sched grid@2 --precision $prec | grep -A6 "rounds \[9"; done
done
} > gpurun_out/${TAG}.txt 2>&1
echo done
