mkdir -p gpurun_out
for a in "256" "256 1024 8"; do
for e in 0 1 2 6 10 14; do SK_EXP=$e timeout 300 python tools/prof_c3.py $a | sed "s/^/exp$e /" >> gpurun_out/exp.log 2>&1; done; done
