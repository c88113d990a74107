mkdir -p gpurun_out
timeout 600 python tools/quick_perf.py > gpurun_out/quick.json 2>&1
