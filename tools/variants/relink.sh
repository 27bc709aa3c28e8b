#!/bin/bash
# Recompile the listed sources of an existing variant and relink it:
#   tools/variants/relink.sh <name> "<-D flags>" fused_pipe [more sources]
set -e
cd "$(dirname "$0")/../../paper_2205_02990_b200/csrc"
name=$1; flags=$2; shift 2
for f in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -c $f.cu -o build_v/$name/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/$name.so build_v/$name/*.o -lcudart
