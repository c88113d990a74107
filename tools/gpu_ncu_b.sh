mkdir -p gpurun_out
SK_EXP=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_bwd_mma" -c 1 -o gpurun_out/bwdB16 python tools/prof_c3.py 128 > gpurun_out/ncu_bwdB16.log 2>&1
