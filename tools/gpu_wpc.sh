mkdir -p gpurun_out
for w in 1 2; do
SK_BWD_WPC=$w timeout 300 python tools/prof_c3.py 256 1024 8 | sed "s/^/wpc$w /" >> gpurun_out/wpc.log 2>&1
SK_BWD_WPC=$w timeout 300 python tools/prof_c3.py 256 | sed "s/^/wpc$w /" >> gpurun_out/wpc.log 2>&1
done
