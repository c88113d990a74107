mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_mma_gpu.py tests/test_forward_gpu.py tests/test_backward_gpu.py -q -x -m gpu > gpurun_out/t32.log 2>&1
for e in 0 1; do SK_NO_MMA=$e python tools/prof_fwd.py 512 512 32 >> gpurun_out/t32.log 2>&1; SK_NO_MMA=$e python tools/prof_fwd.py 512 512 24 >> gpurun_out/t32.log 2>&1; done
