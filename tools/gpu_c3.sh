# C3 headline kernel: DMMA parity tests, bench line, DRAM traffic of the fused kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mma_gpu.py tests/test_baseline_shapes_gpu.py tests/test_determinism_gpu.py -q -x -m gpu > gpurun_out/c3_tests.log 2>&1; echo "rc $?" >> gpurun_out/c3_tests.log
timeout 600 python bench.py --no-cpu --steps 3 > gpurun_out/c3_bench.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gram_bwd" -c 1 --csv --log-file gpurun_out/c3_traffic.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
