#!/bin/bash
# C5 stage under library variants (tools/build_variant.sh): FFPS_LIB_VARIANT per run
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
OUT=gpurun_out/${1:-variants}.txt; shift
{
for v in default "$@"; do
  echo "=== variant $v"
  if [ "$v" = default ]; then unset FFPS_LIB_VARIANT; else export FFPS_LIB_VARIANT=$v; fi
  timeout 900 python tools/sweep_strong.py --n 50000 --iters 12500 --batches 16 64 --scheds grid 2>&1
  timeout 900 python tools/sweep_strong.py --n 75000 --iters 18750 --batches 32 --scheds grid --precisions f64 2>&1
done
} > $OUT 2>&1
echo done
