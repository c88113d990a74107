# C2 (RBF batch, 256 pairs, L=256, d=8, lambda=2): GPU parity of the touched kernels + fwd/bwd timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_backward_gpu.py tests/test_baseline_shapes_gpu.py tests/test_determinism_gpu.py tests/test_transforms.py -q -x -m gpu > gpurun_out/c2_tests.log 2>&1; echo "rc $?" >> gpurun_out/c2_tests.log
timeout 600 python tools/time_c2.py > gpurun_out/c2.log 2>&1
