#!/bin/bash
# ncu --set full of one k_residual_single launch (config 3 T7 at 256^2) for two library variants (A/B)
mkdir -p gpurun_out
for v in ${VARIANTS:-off nz}; do
  RR_LIB_VARIANT=build/variants/$v.so timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:k_residual_single -c 1 -o gpurun_out/prof_ab_$v -f python tools/profile_run.py 3 512 0x40 32 \
    > gpurun_out/ncu_ab_$v.log 2>&1; echo "$v ncu exit $?"
done
