mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mma_gpu.py tests/test_forward_gpu.py tests/test_backward_gpu.py tests/test_conformance_gpu.py tests/test_transforms.py tests/test_baseline_shapes_gpu.py -q -x -m gpu > gpurun_out/dy.log 2>&1; echo "rc $?" >> gpurun_out/dy.log
for e in 0 1; do SK_NO_MMA=$e python tools/time_fwd_small.py 2>&1 | grep Gram >> gpurun_out/dy.log; SK_NO_MMA=$e python tools/prof_fwd.py 256 128 8 1 >> gpurun_out/dy.log 2>&1; SK_NO_MMA=$e python tools/prof_fwd.py 256 256 16 2 >> gpurun_out/dy.log 2>&1; done
