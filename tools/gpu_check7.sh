mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest.log | head -20
timeout 300 python -m pytest tests/test_gpu_coverage.py -q --durations=10 2>&1 | tail -14
