# DRAM bytes of the DMMA backward (prof_c3.py n=512) under SK_EXP switches (profiling build)
mkdir -p gpurun_out
export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/prof/libsigkernel.so
for e in 0 4 1; do
  SK_EXP=$e timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"gram_bwd" -c 1 --csv --log-file gpurun_out/tr_exp$e.csv python tools/prof_c3.py 512 > /dev/null 2>&1
done
