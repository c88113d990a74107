mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_mma_gpu.py -q -x -k forward > gpurun_out/fw_tests.log 2>&1
for w in 4 2 1; do
for a in "256 512 16" "256 1024 8"; do SK_FWD_WPC=$w timeout 300 python tools/prof_fwd.py $a | sed "s/^/fwpc$w /" >> gpurun_out/fwpc.log 2>&1; done; done
SK_FWD_WPC=2 timeout 300 python -m pytest tests/test_mma_gpu.py -q -x -k forward >> gpurun_out/fw_tests.log 2>&1
