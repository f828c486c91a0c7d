mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --no-exhaustive --no-cpu-baseline > gpurun_out/bench_q$i.json 2>&1; echo bench=$?
python -c "
import json;d=json.load(open('gpurun_out/bench_q$i.json'))
print(d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['step_ms'], d['clocks'])"
done
