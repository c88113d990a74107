mkdir -p gpurun_out
for e in 0 1; do echo "== SK_NO_MMA=$e" >> gpurun_out/dy2.log; for a in "256 128 16 1" "256 128 32 1" "256 128 8 1" "256 64 16 2" "256 128 4 1"; do SK_NO_MMA=$e python tools/prof_fwd.py $a >> gpurun_out/dy2.log 2>&1; done; done
