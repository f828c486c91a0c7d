mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest.log | grep -vE "^\s*$" | tail -12
timeout 600 python tools/sweep.py --batch 64 --n 50000 --cloud-n 200000 --iters 12500 --plans 256,14,36,4 128,28,72,4 128,10,36,9 256,8,20,7 256,4,16,10 512,14,36,2 256,16,24,5 > gpurun_out/sweep_flash.jsonl 2>&1; echo sweep=$?
cat gpurun_out/sweep_flash.jsonl
timeout 600 python tools/sweep.py --batch 64 --n 200000 --iters 50000 --reps 1 --plans 128,28,72,16 256,14,36,16 512,14,36,8 > gpurun_out/sweep_exh.jsonl 2>&1; echo sweep2=$?
cat gpurun_out/sweep_exh.jsonl
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
