# forward DMMA check: parity tests, old-vs-new timings, ncu of the new kernel
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mma_gpu.py tests/test_forward_gpu.py tests/test_conformance_gpu.py -x -q > gpurun_out/fwd_tests.log 2>&1; echo "rc $?" >> gpurun_out/fwd_tests.log
for args in "1024 512 16" "512 1024 8" "256 512 16"; do
  timeout 300 python tools/prof_fwd.py $args >> gpurun_out/fwd_perf.log 2>&1
  SK_NO_MMA=1 timeout 300 python tools/prof_fwd.py $args | sed 's/^/old /' >> gpurun_out/fwd_perf.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gram_fwd_mma" -c 1 -o gpurun_out/fwd_mma python tools/prof_fwd.py 256 512 16 > gpurun_out/ncu_fwd_mma.log 2>&1
