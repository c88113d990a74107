mkdir -p gpurun_out
for e in 1 0; do echo "== SK_MMA_PST=$e" >> gpurun_out/pst.log; SK_MMA_PST=$e python tools/prof_c3.py 512 >> gpurun_out/pst.log 2>&1; SK_MMA_PST=$e python tools/prof_c3.py 512 1024 8 >> gpurun_out/pst.log 2>&1; done
timeout 900 python -m pytest tests/test_mma_gpu.py tests/test_baseline_shapes_gpu.py tests/test_determinism_gpu.py -q -x -m gpu 2>&1 | tail -2 >> gpurun_out/pst.log
