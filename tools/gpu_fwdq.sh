mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mma_gpu.py tests/test_forward_gpu.py -x -q > gpurun_out/fwd_tests.log 2>&1; echo "rc $?" >> gpurun_out/fwd_tests.log
for a in "256 512 16" "256 1024 8"; do timeout 300 python tools/prof_fwd.py $a >> gpurun_out/fwd_perf.log 2>&1; done
