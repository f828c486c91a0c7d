mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo pytest=$?
grep -E "passed|failed|Error|assert" gpurun_out/pytest.log | head -20
for PIPE in 1 0; do
 for CL in 200000; do
  FFPS_BUCKET_PIPE=$PIPE FFPS_ALGO=bucket timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n $CL --iters 12500 --reps 3 2>&1 | tail -1
  FFPS_BUCKET_PIPE=$PIPE FFPS_ALGO=bucket timeout 600 python tools/sweep.py --batch 64 --n 200000 --iters 50000 --reps 2 2>&1 | tail -1
 done
done
