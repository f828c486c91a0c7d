#!/bin/bash
# round 2, first GPU session: smoke, new parity tests, bench (binary64 headline), strong-scaling sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r02a_smoke.txt
timeout 900 python -m pytest tests/test_gpu_mixed.py tests/test_gpu_api_edges.py -x -q > gpurun_out/r02a_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/r02a_tests.txt
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?" >> gpurun_out/r02a_bench.err
timeout 600 python tools/sweep_strong.py > gpurun_out/r02a_strong.jsonl 2>&1
echo done
