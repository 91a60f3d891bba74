#!/bin/bash
# Phase-timer profile of the engine at two moves-per-round settings (bench window).
O=gpurun_out/$1; mkdir -p $O
for cfg in "prof256 256" "prof512 128"; do
  set -- $cfg
  echo "== lib $1 group $2" >> $O/prof.log
  env GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$1.so GCMC_ENGINE_GROUP=$2 GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 1048576 --warm 12582912 >> $O/prof.log 2>&1
done
