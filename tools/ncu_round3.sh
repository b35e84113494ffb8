#!/bin/bash
# ncu evidence after the symv/GEMM changes (measurement tool): each command runs plain
# first, then one --set full capture of the kernel in situ.
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --set full --clock-control none --import-source on"
# the in-sytrd symv (dlarfg + quadratic-form instantiation), ~column 40 of panel 0 at N=16k
python tools/prof_kernels.py syev > $OUT/r3_plain_syev.json 2>&1 && \
  $NCU -k regex:symv_tma_kernel -s 40 -c 1 -o $OUT/r3_ncu_symv_sytrd python tools/prof_kernels.py syev > $OUT/r3_ncu_symv.log 2>&1
# the 64x64-tile GEMM on 8192^3
python tools/prof_kernels.py gemm > $OUT/r3_plain_gemm.json 2>&1 && \
  $NCU -k regex:gemm_kernel -s 1 -c 1 -o $OUT/r3_ncu_gemm python tools/prof_kernels.py gemm > $OUT/r3_ncu_gemm.log 2>&1
# the C5-shaped replay
export TD2_N=60000 TD2_T=100000 TD2_OBS=64
python tools/prof_kernels.py td2 > $OUT/r3_plain_td2.json 2>&1 && \
  $NCU -k regex:td2_replay -s 1 -c 1 -o $OUT/r3_ncu_td2_replay python tools/prof_kernels.py td2 > $OUT/r3_ncu_td2.log 2>&1
echo done
