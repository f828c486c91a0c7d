mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 500 > gpurun_out/clk.csv &)
for cfg in "0 0" "0 1" "1 1" "1 0"; do
  set -- $cfg
  echo "PIPE=$1 SORT2=$2"
  FFPS_BUCKET_PIPE=$1 FFPS_BUCKET_SORT2=$2 FFPS_ALGO=bucket timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --reps 5 2>&1 | tail -1
done
sort gpurun_out/clk.csv | uniq -c | sort -rn | head -5
