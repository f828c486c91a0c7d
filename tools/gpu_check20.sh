mkdir -p gpurun_out
timeout 300 python tools/trace_multi.py --sched grid@2
timeout 300 python tools/trace_multi.py --sched grid@1
