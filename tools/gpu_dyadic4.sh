mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dy4.log 2>&1; echo "rc $?" >> gpurun_out/dy4.log
for a in "512 256 4 0" "512 256 8 0" "256 128 8 1" "256 128 16 1" "256 128 32 1"; do python tools/prof_fwd.py $a >> gpurun_out/dy4.log 2>&1; done
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/dy4.log 2>&1
