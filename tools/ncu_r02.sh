#!/bin/bash
# Round-2 ncu evidence (measurement tool): each workload runs plain first, then one
# --set full capture of the kernel in situ (one GPU, never multi-rank).
#   bash tools/ncu_r02.sh [q2|trsv|gemm|all]
set -u
OUT=gpurun_out
mkdir -p $OUT
WHAT=${1:-all}
NCU="ncu --set full --clock-control none --import-source on"
if [ "$WHAT" = q2 ] || [ "$WHAT" = all ]; then
  # register-resident Q2 back-transform, n = 16384 (group ~155 of the first em_syev: 101 blocks)
  python tools/q2_probe.py 16384 0 > $OUT/r02_plain_q2.log 2>&1 && \
    $NCU -k regex:q2r_kernel -s 100 -c 1 -o $OUT/r02_ncu_q2r python tools/q2_probe.py 16384 0 \
      > $OUT/r02_ncu_q2r.log 2>&1
fi
if [ "$WHAT" = trsv ] || [ "$WHAT" = all ]; then
  # the TD1 triangular solves at N = 16384 (steps 10 and 11 of the timed run)
  export TD1_N=16384
  python tools/prof_kernels.py td1 > $OUT/r02_plain_td1.json 2>&1 && \
    $NCU -k regex:trsv_ -s 20 -c 2 -o $OUT/r02_ncu_trsv python tools/prof_kernels.py td1 \
      > $OUT/r02_ncu_trsv.log 2>&1
fi
if [ "$WHAT" = gemm ] || [ "$WHAT" = all ]; then
  python tools/prof_kernels.py gemm > $OUT/r02_plain_gemm.json 2>&1 && \
    $NCU -k regex:gemm_kernel -s 1 -c 1 -o $OUT/r02_ncu_gemm python tools/prof_kernels.py gemm \
      > $OUT/r02_ncu_gemm.log 2>&1
fi
echo done
