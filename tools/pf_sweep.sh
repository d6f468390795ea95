#!/bin/bash
# Kernel time vs the prologue-time L2 prefetch depth (RSR_MV_PF rounds).
for pf in ${1:-0 2 4 8 12}; do
  echo "pf=$pf"; RSR_MV_PF=$pf tools/mv_ncu_experiments.sh "0" ${2:-float} 2>&1 | grep gpu__time
done
