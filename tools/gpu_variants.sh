mkdir -p gpurun_out
for v in base cb32 cb64; do
  if [ $v = base ]; then unset SK_LIBSIGKERNEL; else export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/$v/libsigkernel.so; fi
  echo "== $v" >> gpurun_out/v.log
  python tools/time_c2.py 1 >> gpurun_out/v.log 2>&1
  python tools/time_c2.py 0 >> gpurun_out/v.log 2>&1
done
export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/cb32/libsigkernel.so
timeout 600 python -m pytest tests/test_backward_gpu.py tests/test_baseline_shapes_gpu.py -q -x -m gpu 2>&1 | tail -2 >> gpurun_out/v.log
