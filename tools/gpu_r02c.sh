#!/bin/bash
# new GPU suites of round 2: full-shape parity, reference-suite replay, verify port, PNN adapter
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nproc > gpurun_out/r02c_nproc.txt
timeout 1500 python -m pytest tests/test_gpu_reference_suite.py tests/test_gpu_verify.py tests/test_gpu_pnn.py tests/test_gpu_api_edges.py -q -s --durations=15 > gpurun_out/r02c_suites.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c_suites.txt
timeout 2400 python -m pytest tests/test_gpu_fullscale.py -q --durations=20 > gpurun_out/r02c_fullscale.txt 2>&1; echo "rc=$?" >> gpurun_out/r02c_fullscale.txt
echo done
