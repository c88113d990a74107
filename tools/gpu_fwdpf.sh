mkdir -p gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then unset SK_LIBSIGKERNEL; else export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/$v/libsigkernel.so; fi
  echo "== $v" >> gpurun_out/pf.log
  python tools/time_fwd_small.py >> gpurun_out/pf.log 2>&1
  python tools/time_c2.py 1 >> gpurun_out/pf.log 2>&1
done
unset SK_LIBSIGKERNEL
timeout 900 python -m pytest tests/test_forward_gpu.py tests/test_baseline_shapes_gpu.py tests/test_conformance_gpu.py tests/test_fp32_gpu.py tests/test_transforms.py -q -x -m gpu 2>&1 | tail -2 >> gpurun_out/pf.log
