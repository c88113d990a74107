mkdir -p gpurun_out
for e in 0 1; do echo "== SK_NO_MMA=$e" >> gpurun_out/dy3.log; for a in "512 256 4 0" "512 256 8 0" "256 128 2 1"; do SK_NO_MMA=$e python tools/prof_fwd.py $a >> gpurun_out/dy3.log 2>&1; done; done
