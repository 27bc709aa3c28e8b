#!/bin/bash
# Builds a tracing variant of the library into tools/trace/_hbs_b200_trace.so
set -e
cd "$(dirname "$0")/../../paper_2205_02990_b200/csrc"
mkdir -p build_trace
for f in hqr cholqr applyq applyq2 bgemm capi sampler; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DHBS_TRACE $EXTRA -c $f.cu -o build_trace/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/trace/_hbs_b200_trace.so build_trace/*.o -lcudart
