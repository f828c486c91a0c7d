#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_scale.py -q -x -k "host" 2>&1 | tail -1
FFPS_E2E_ZEROCOPY=1 timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_scale.py -q -x -k "host" 2>&1 | tail -1
echo "-- staged"; FFPS_E2E_PRECISION=f64 timeout 600 python tools/e2e_chunks.py 1 2 4
echo "-- zero-copy"; FFPS_E2E_ZEROCOPY=1 FFPS_E2E_PRECISION=f64 timeout 600 python tools/e2e_chunks.py 1 2 4 8
} > gpurun_out/e2e.txt 2>&1
echo done
