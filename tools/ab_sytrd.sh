set -e
for v in new old noshift; do
  unset EM_LIB_PATH SYTRD_DBG
  if [ $v = old ]; then export EM_LIB_PATH=$PWD/build/old_4ae9aac.so; fi
  if [ $v = noshift ]; then export SYTRD_DBG=16; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 300 --launch-count 120 --csv --log-file gpurun_out/ab_$v.csv python tools/prof_kernels.py syev > /dev/null 2>&1
done
