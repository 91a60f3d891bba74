#!/bin/bash
# A/B of engine builds/env settings on one box: each argument is an env
# assignment list ("" = default), e.g.  bash tools/gpu_envab.sh TAG "" "GCMC_WALK_REPS=7"
O=gpurun_out/${1:-envab}; mkdir -p $O; shift
i=0
for e in "$@"; do
  env $e timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 > $O/ab$i.log 2>&1
  echo "[$e]: $(tail -1 $O/ab$i.log)" >> $O/summary.txt
  i=$((i+1))
done
