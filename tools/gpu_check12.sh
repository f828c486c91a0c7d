mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest.log | head -20
for A in grid bucket; do
FFPS_ALGO=$A timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --reps 5 2>&1 | tail -1 | cut -c1-100
FFPS_ALGO=$A timeout 600 python tools/sweep.py --batch 64 --n 200000 --iters 50000 --reps 2 2>&1 | tail -1 | cut -c1-100
done
timeout 300 python tools/trace_multi.py --sched grid
