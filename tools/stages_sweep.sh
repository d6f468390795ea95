for st in 2 4 6 8; do RSR_MV_STAGES=$st tools/mv_ncu_experiments.sh "0 32" float | sed "s/^/S=$st /"; done
