#!/bin/bash
# One GPU call: plain runs, then ncu captures of the hot kernels (each command ran
# plain first, as the profiling recipe requires), then the launch list of a C1 bench.
set -u
OUT=gpurun_out
mkdir -p $OUT
for k in symv gemm td2 td1; do
  python tools/prof_kernels.py $k > $OUT/prof_plain_$k.json 2>> $OUT/prof_plain.err || exit 3
done
NCU="ncu --set full --clock-control none --import-source on"
python tools/prof_kernels.py symv > /dev/null && \
  $NCU -k regex:symv_tiles -s 2 -c 1 -o $OUT/ncu_symv python tools/prof_kernels.py symv > $OUT/ncu_symv.log 2>&1
python tools/prof_kernels.py gemm > /dev/null && \
  $NCU -k regex:gemm_kernel -s 1 -c 1 -o $OUT/ncu_gemm python tools/prof_kernels.py gemm > $OUT/ncu_gemm.log 2>&1
python tools/prof_kernels.py td2 > /dev/null && \
  $NCU -k regex:td2_replay -s 1 -c 1 -o $OUT/ncu_td2 python tools/prof_kernels.py td2 > $OUT/ncu_td2.log 2>&1
python tools/prof_kernels.py td1 > /dev/null && \
  $NCU -k regex:"trsv_(fwd|bwd)" -s 20 -c 2 -o $OUT/ncu_td1 python tools/prof_kernels.py td1 > $OUT/ncu_td1.log 2>&1
python bench.py --config C1 --steps 1 --warmup 3 --no-e2e --no-td1 --no-cpu > $OUT/launch_plain.json 2>/dev/null && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file $OUT/launches_c1.csv \
    python bench.py --config C1 --steps 1 --warmup 3 --no-e2e --no-td1 --no-cpu > $OUT/launch_ncu.log 2>&1
echo done
