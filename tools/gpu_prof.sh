# ncu --set full captures: C2 RBF batch forward + backward (current build), C3 DMMA backward at n=512
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_kernel" -c 2 -o gpurun_out/c2_fb python tools/prof_c2.py fb > gpurun_out/ncu_c2.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"gram_bwd_mma" -c 1 -o gpurun_out/c3_512 python tools/prof_c3.py 512 > gpurun_out/ncu_c3.log 2>&1
