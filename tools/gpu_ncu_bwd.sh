mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_bwd_mma" -c 1 -o gpurun_out/bwd_mma16 python tools/prof_c3.py 128 > gpurun_out/ncu_bwd16.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_bwd_mma" -c 1 -o gpurun_out/bwd_mma8 python tools/prof_c3.py 128 1024 8 > gpurun_out/ncu_bwd8.log 2>&1
