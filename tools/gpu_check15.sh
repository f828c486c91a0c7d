mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid" 2>&1 | tail -1
for shape in "64 50000 12500 200000" "64 200000 50000 200000" "8 100000 25000 100000" "32 75000 18750 300000"; do
  set -- $shape
  r=$(FFPS_ALGO=grid timeout 600 python tools/sweep.py --batch $1 --n $2 --iters $3 --cloud-n $4 --reps 3 2>&1 | tail -1 | python -c "import json,sys;print(json.load(sys.stdin)['ms'])")
  echo "grid B=$1 n=$2 iters=$3 ms=$r"
done
timeout 300 python tools/trace_multi.py --sched grid
