# C2 RBF backward with the epilogue ILP variants (tools/build_variant.sh epiA / epiB)
V=paper_2509_10613_b200/_native/variants
for i in 1 2; do
for lib in base epiA epiB; do
  if [ $lib = base ]; then unset SK_LIBSIGKERNEL; else export SK_LIBSIGKERNEL=$V/$lib/libsigkernel.so; fi
  echo "== $lib"; python tools/time_c2.py 1 2>&1 | tail -1
done; done
for lib in epiA epiB; do
  SK_LIBSIGKERNEL=$V/$lib/libsigkernel.so timeout 300 python -m pytest tests/test_backward_gpu.py tests/test_baseline_shapes_gpu.py tests/test_determinism_gpu.py -q -x 2>&1 | tail -1
done
