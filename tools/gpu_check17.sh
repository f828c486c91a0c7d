# e2e with whole-batch cluster size + LiDAR K1g traces
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --exh-steps 1 > gpurun_out/bench17.json 2> gpurun_out/bench17.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench17.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], d["roofline"]["kernel"])
PY
for s in grid@1 grid@2; do
  echo "== lidar $s"; timeout 300 python tools/trace_multi.py --sched $s --cloud lidar
done
FFPS_ALGO=bucket timeout 300 python tools/sweep.py --batch 64 --n 50000 --iters 12500 --cloud-n 200000 --reps 3 2>&1 | tail -1
