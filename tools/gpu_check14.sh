mkdir -p gpurun_out
for KM in 8 16; do
for shape in "64 50000 12500 200000" "64 200000 50000 200000" "8 100000 25000 100000" "32 75000 18750 300000" "32 300000 75000 300000"; do
  set -- $shape
  r=$(FFPS_GRID_KM=$KM FFPS_ALGO=grid timeout 600 python tools/sweep.py --batch $1 --n $2 --iters $3 --cloud-n $4 --reps 3 2>&1 | tail -1 | python -c "import json,sys;print(json.load(sys.stdin)['ms'])")
  echo "KM=$KM B=$1 n=$2 iters=$3 ms=$r"
done
done
