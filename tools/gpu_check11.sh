mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "multi or schedule" 2>&1 | tail -1
for A in multi bucket; do
FFPS_ALGO=$A timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --reps 5 2>&1 | tail -1 | cut -c1-120
done
timeout 300 python tools/trace_multi.py
