# time the C3 step (prof_c3.py at n given) under SK_EXP switches of the profiling build
mkdir -p gpurun_out
export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/prof/libsigkernel.so
for e in 0 8 4 1; do
  echo "== SK_EXP=$e" >> gpurun_out/exp.log
  SK_EXP=$e python tools/prof_c3.py ${1:-512} >> gpurun_out/exp.log 2>&1
done
