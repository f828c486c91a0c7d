#!/bin/bash
# debug-checked library (device asserts on shared-memory list bounds) under the parity suites, + fused hierarchy
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
echo "=== default library: new tests"
timeout 900 python -m pytest tests/test_gpu_mixed.py -q -k fused 2>&1 | tail -2
echo "=== FFPS_LIB_VARIANT=checks (-DFFPS_DEBUG_CHECKS)"
export FFPS_LIB_VARIANT=checks
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_gpu_scale.py tests/test_gpu_coverage.py -q -x 2>&1 | tail -3
} > gpurun_out/r02e.txt 2>&1
echo done
