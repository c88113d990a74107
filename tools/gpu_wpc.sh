mkdir -p gpurun_out
for w in 2 3 4; do echo "== SK_BWD_WPC=$w" >> gpurun_out/wpc.log; SK_BWD_WPC=$w python tools/prof_c3.py 512 >> gpurun_out/wpc.log 2>&1; SK_BWD_WPC=$w python tools/prof_c3.py 512 1024 8 >> gpurun_out/wpc.log 2>&1; done
