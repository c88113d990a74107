mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_mma_gpu.py -q -x -m gpu > gpurun_out/dyb.log 2>&1; echo "rc $?" >> gpurun_out/dyb.log
timeout 900 python -m pytest tests -m gpu -x -q >> gpurun_out/dyb.log 2>&1; echo "all rc $?" >> gpurun_out/dyb.log
for v in "0" "1"; do for a in "256 129 16 1" "256 129 12 1" "256 65 16 2" "256 129 8 1"; do SK_MMA_DY=$v python tools/prof_bwd_dy.py $a >> gpurun_out/dyb.log 2>&1; done; done
