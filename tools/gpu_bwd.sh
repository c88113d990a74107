mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mma_gpu.py -x -q > gpurun_out/bwd_tests.log 2>&1; echo "rc $?" >> gpurun_out/bwd_tests.log
for a in "256" "256 1024 8"; do
for e in 0 1 2; do SK_EXP=$e timeout 300 python tools/prof_c3.py $a | sed "s/^/exp$e /" >> gpurun_out/bwd_perf.log 2>&1; done; done
