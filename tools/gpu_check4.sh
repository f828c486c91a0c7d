mkdir -p gpurun_out
set -x
timeout 1200 python -m pytest tests -m gpu -q --maxfail=8 -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest.log | head -30
for A in bucket stream; do
FFPS_ALGO=$A timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --reps 3 2>&1 | tail -1
done > gpurun_out/sweep_flash_algo.jsonl
cat gpurun_out/sweep_flash_algo.jsonl
FFPS_ALGO=bucket timeout 600 python tools/sweep.py --batch 64 --n 200000 --iters 50000 --reps 2 2>&1 | tail -1 > gpurun_out/sweep_exh_bucket.jsonl
cat gpurun_out/sweep_exh_bucket.jsonl
