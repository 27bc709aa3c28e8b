#!/bin/bash
# builds panel_bench variants for the step ablation (development tool)
cd "$(dirname "$0")"
B=../../paper_2205_02990_b200/csrc/build
for v in ${VARIANTS:-BASE PF_EXP_NOREFL PF_EXP_NOPUB PF_EXP_NONEED}; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -diag-suppress 177 \
    $(echo -D$v | sed "s/+/ -D/g") -DPB_NBP=${NBP:-32} -I../../paper_2205_02990_b200/csrc panel_bench.cu $B/capi.o $B/applyq.o $B/applyq2.o $B/bgemm.o \
    $B/sampler.o -o pb_${v//+/_} &
done
wait
