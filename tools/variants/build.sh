#!/bin/bash
# Builds library variants tools/variants/<name>.so from "name:FLAGS" specs
# (FLAGS comma-separated -D macros), for A/B timing with HBS_B200_LIB.
set -e
cd "$(dirname "$0")/../../paper_2205_02990_b200/csrc"
for spec in "$@"; do
  name=${spec%%:*}; flags=$(echo "${spec#*:}" | tr ',' ' ')
  (mkdir -p build_v/$name
   for f in hqr fused_pipe fused_split gram gram_tm cholqr applyq applyq2 bgemm capi sampler; do
     nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -c $f.cu -o build_v/$name/$f.o &
   done
   wait; nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/variants/$name.so build_v/$name/*.o -lcudart) &
done
wait
