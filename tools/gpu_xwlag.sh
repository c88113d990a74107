V=paper_2509_10613_b200/_native/variants
for i in 1 2; do
for lib in base lag8 lag2; do
  if [ $lib = base ]; then unset SK_LIBSIGKERNEL; else export SK_LIBSIGKERNEL=$V/$lib/libsigkernel.so; fi
  echo "== $lib"; python tools/time_c2.py 1 2>&1 | tail -2; python tools/time_c4.py 2>&1 | tail -1
done; done
unset SK_LIBSIGKERNEL
SK_LIBSIGKERNEL=$V/lag8/libsigkernel.so timeout 300 python -m pytest tests/test_forward_gpu.py tests/test_baseline_shapes_gpu.py -q -x 2>&1 | tail -1
