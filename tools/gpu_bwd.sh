mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mma_gpu.py -x -q > gpurun_out/bwd_tests.log 2>&1; echo "rc $?" >> gpurun_out/bwd_tests.log
timeout 300 python tools/prof_c3.py 256 > gpurun_out/bwd_perf.log 2>&1
SK_NO_MMA=1 timeout 300 python tools/prof_c3.py 256 | sed 's/^/old /' >> gpurun_out/bwd_perf.log 2>&1
timeout 300 python tools/prof_c3.py 256 1024 8 >> gpurun_out/bwd_perf.log 2>&1
SK_NO_MMA=1 timeout 300 python tools/prof_c3.py 256 1024 8 | sed 's/^/old /' >> gpurun_out/bwd_perf.log 2>&1
