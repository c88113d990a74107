# C3-shape DMMA backward (prof_c3.py n=512) for the in-tree build and the named variants
mkdir -p gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then unset SK_LIBSIGKERNEL; else export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/$v/libsigkernel.so; fi
  echo "== $v" >> gpurun_out/c3var.log
  python tools/prof_c3.py 512 >> gpurun_out/c3var.log 2>&1
  python tools/prof_c3.py 512 >> gpurun_out/c3var.log 2>&1
done
