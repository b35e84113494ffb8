#!/bin/bash
# Round-1 refresh of the ncu evidence (measurement tool): each command runs plain first
# (the profiling recipe), then one --set full capture of the kernel, then the launch list
# of a C1 bench step.
set -u
OUT=gpurun_out
mkdir -p $OUT
NCU="ncu --set full --clock-control none --import-source on"
export TD2_OBS=64
python tools/prof_kernels.py td2 > $OUT/prof_plain_td2.json 2>&1 && \
  $NCU -k regex:td2_replay -s 1 -c 1 -o $OUT/ncu_td2_replay python tools/prof_kernels.py td2 > $OUT/ncu_td2.log 2>&1
python tools/prof_kernels.py symv > $OUT/prof_plain_symv.json 2>&1 && \
  $NCU -k regex:symv_tma_kernel -s 2 -c 1 -o $OUT/ncu_symv python tools/prof_kernels.py symv > $OUT/ncu_symv.log 2>&1
python tools/prof_kernels.py gemm > $OUT/prof_plain_gemm.json 2>&1 && \
  $NCU -k regex:gemm_kernel -s 1 -c 1 -o $OUT/ncu_gemm python tools/prof_kernels.py gemm > $OUT/ncu_gemm.log 2>&1
python bench.py --config C1 --steps 1 --warmup 3 --no-e2e --no-td1 --no-cpu > $OUT/launch_plain.json 2>/dev/null && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_c1.csv \
    python bench.py --config C1 --steps 1 --warmup 3 --no-e2e --no-td1 --no-cpu > $OUT/launch_ncu.log 2>&1
echo done
