mkdir -p gpurun_out
set -x
# per-iteration latency floor: tiny clouds, one cluster, sizes C = 1..16
for C in 1 2 4 8 16; do
  python tools/sweep.py --batch 1 --n $((512*C)) --iters 20000 --reps 3 --plans 256,2,0,$C 128,2,0,$C 2>&1 | tail -2
done > gpurun_out/lat.jsonl
cat gpurun_out/lat.jsonl
# work scaling at fixed C=4: per-iteration time vs points per CTA
for P in "256,2,0" "256,8,0" "256,16,0" "256,16,8" "256,16,24" "256,14,36"; do
  IFS=, read nt p s <<< "$P"; n=$((nt*(p+s)*4))
  python tools/sweep.py --batch 1 --n $n --iters 5000 --reps 3 --plans $P,4 2>&1 | tail -1
  python tools/sweep.py --batch 64 --n $n --iters 5000 --reps 3 --plans $P,4 2>&1 | tail -1
done > gpurun_out/work.jsonl
cat gpurun_out/work.jsonl
C1="python tools/sweep.py --batch 64 --n 50000 --cloud-n 50000 --iters 2000 --reps 1"
$C1 > gpurun_out/c1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fps_greedy -s 1 -c 1 -o gpurun_out/prof_k1v2 $C1 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
