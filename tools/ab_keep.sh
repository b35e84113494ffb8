# A/B of EM_CFG_SYMV_L2_KEEP_MB on the sytrd stage (em_syev at SYEV_N, stage timers)
set -e
for k in ${KEEPS:-0 80 0 40 80 110}; do
  echo "keep=$k $(SYMV_KEEP_MB=$k python tools/prof_kernels.py syev | python -c 'import json,sys; d=json.load(sys.stdin); print({k:v for k,v in d.items() if "level1" in k})')"
done
