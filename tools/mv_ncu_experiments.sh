#!/bin/bash
# Device-side kernel durations (ncu gpu__time_duration) of the multiply under
# the RSR_MV_DEBUG experiment knobs.  usage: tools/mv_ncu_experiments.sh "0 32 64" [float|int] [cfg] [k]
KNOBS=${1:-"0"}
MODE=${2:-float}
CFG=${3:-c2}
K=${4:-6}
for d in $KNOBS; do
  RSR_B200_LIB=${RSR_B200_LIB:-} RSR_MV_DEBUG=$d python tools/profile_matvec.py $CFG $K $MODE 4 > /dev/null 2>&1 || { echo "plain run failed dbg=$d"; continue; }
  RSR_MV_DEBUG=$d ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:rsr_mv -s 1 -c 3 --csv python tools/profile_matvec.py $CFG $K $MODE 4 2>/dev/null \
    | grep -E "gpu__time_duration|dram__bytes_read" | awk -F'","' -v d=$d -v m=$MODE '{gsub(/"/,"",$NF); print m, "dbg="d, $(NF-2), $NF}'
done
