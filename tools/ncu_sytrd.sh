#!/bin/bash
# Launch lists (ncu gpu__time_duration) of three tridiagonalisation panels at N=8192:
# panel 0 (m ~ 8192), panel 64 (m ~ 4096), panel 112 (m ~ 1024). Measurement tool.
set -e
mkdir -p gpurun_out
export SYEV_N=${SYEV_N:-8192}
PER=${PER:-455}
for p in ${PANELS:-0 64 112}; do
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip $((p * PER)) \
      --launch-count $PER --csv --log-file gpurun_out/sytrd_p${p}.csv \
      python tools/prof_kernels.py syev > /dev/null 2>&1
done
