mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python tools/prof_c3.py 256 1024 8 | sed 's/fwd.*bwd/bwd/' >> gpurun_out/rep.log; timeout 300 python tools/prof_c3.py 256 | sed 's/fwd.*bwd/bwd/' >> gpurun_out/rep.log; done
