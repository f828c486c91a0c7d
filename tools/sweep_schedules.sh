# every schedule on the greedy stage shapes of the BASELINE configs
mkdir -p gpurun_out
run() {  # B n iters cloud_n
  for A in stream bucket multi grid; do
    if [ "$A" = stream ] && [ "$2" -ge 200000 ]; then R=1; else R=3; fi
    r=$(FFPS_ALGO=$A timeout 600 python tools/sweep.py --batch $1 --n $2 --iters $3 --cloud-n $4 --reps $R 2>/dev/null | tail -1 | python -c "import json,sys;print(json.load(sys.stdin)['ms'])")
    echo "{\"B\": $1, \"n\": $2, \"iters\": $3, \"schedule\": \"$A\", \"ms\": $r}"
  done
}
run 16 6000 1500 24000
run 16 24000 6000 24000
run 8 25000 6250 100000
run 8 100000 25000 100000
run 32 75000 18750 300000
run 32 300000 75000 300000
run 64 50000 12500 200000
run 64 200000 50000 200000
run 1 4096 1024 4096
