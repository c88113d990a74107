# time C2 (RBF, linear) and C4 under env settings given as arguments ("VAR=value"
# each; "base" = none), then the forward/backward parity tests under the last one
mkdir -p gpurun_out
for kv in "$@"; do
  echo "== $kv" >> gpurun_out/env.log
  e=""; [ "$kv" != base ] && e="$kv"
  env $e python tools/time_c2.py 1 >> gpurun_out/env.log 2>&1
  env $e python tools/time_c2.py 0 >> gpurun_out/env.log 2>&1
  env $e python tools/time_c4.py >> gpurun_out/env.log 2>&1
done
last="${@: -1}"; e=""; [ "$last" != base ] && e="$last"
env $e timeout 900 python -m pytest tests/test_backward_gpu.py tests/test_forward_gpu.py tests/test_baseline_shapes_gpu.py -q -x -m gpu 2>&1 | tail -2 >> gpurun_out/env.log
