mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest.log | head -20
for shape in "64 50000 12500 200000" "64 200000 50000 200000" "8 100000 25000 100000" "32 75000 18750 300000"; do
  set -- $shape
  FFPS_ALGO=grid timeout 600 python tools/sweep.py --batch $1 --n $2 --iters $3 --cloud-n $4 --reps 3 2>&1 | tail -1 | cut -c1-60
done
timeout 300 python tools/trace_multi.py --sched grid
