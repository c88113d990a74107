#!/bin/bash
# Build an experiment variant of the backward TU into _native/variants/<name>/libsigkernel.so
# usage: tools/build_variant.sh <name> <extra nvcc flags...>
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_2509_10613_b200/_native/variants/$name
mkdir -p $out
objs=""
for src in sk_capi sk_fwd_linear sk_fwd_rbf sk_fwd_delta sk_bwd_rbf; do objs="$objs paper_2509_10613_b200/_native/$src.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ccbin /usr/bin/g++ "$@" -c paper_2509_10613_b200/csrc/sk_bwd_linear.cu -o $out/sk_bwd_linear.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libsigkernel.so $objs $out/sk_bwd_linear.o -lcudart
echo $out/libsigkernel.so
