mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fp32_gpu.py tests/test_transforms.py tests/test_mma_gpu.py -q -x -m gpu > gpurun_out/f32.log 2>&1; echo "rc $?" >> gpurun_out/f32.log
for e in 0 1; do echo "== SK_NO_MMA=$e" >> gpurun_out/f32.log; for a in "1024 512 16 0" "512 1024 8 0" "512 256 4 0" "256 128 16 1" "256 128 8 1"; do SK_NO_MMA=$e python tools/prof_fwd32.py $a >> gpurun_out/f32.log 2>&1; done; done
