# time C2 / C4 for each (library variant, env) pair: args "variant:VAR=value" ("base" = in-tree build, "-" = no env)
mkdir -p gpurun_out
for a in "$@"; do
  v=${a%%:*}; kv=${a#*:}; [ "$kv" = "-" ] && kv=""
  if [ $v = base ]; then unset SK_LIBSIGKERNEL; else export SK_LIBSIGKERNEL=$PWD/paper_2509_10613_b200/_native/variants/$v/libsigkernel.so; fi
  echo "== $v $kv" >> gpurun_out/le.log
  env $kv python tools/time_c2.py 1 >> gpurun_out/le.log 2>&1
  env $kv python tools/time_c2.py 0 >> gpurun_out/le.log 2>&1
  env $kv python tools/time_c4.py >> gpurun_out/le.log 2>&1
done
