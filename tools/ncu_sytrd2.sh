#!/bin/bash
# Launch lists (ncu gpu__time_duration, serialised) of tridiagonalisation panels of
# em_syev at N=16384: the first panels (m ~ N) and a middle stretch (m ~ N/2).
# Measurement tool.
set -e
mkdir -p gpurun_out
export SYEV_N=${SYEV_N:-16384}
python tools/prof_kernels.py syev > gpurun_out/syev_plain.json 2>&1
for sk in 0 ${MID:-26000}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip $sk \
      --launch-count ${CNT:-700} --csv --log-file gpurun_out/sytrd_s${sk}.csv \
      python tools/prof_kernels.py syev > /dev/null 2>&1
done
