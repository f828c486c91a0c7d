# round verification of HEAD: smoke, GPU parity suite, headline bench, reference arm
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref=$?
