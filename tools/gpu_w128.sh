#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for lib in libgcmc_b200.so libgcmc_b200_w128.so; do
 for g in 256 128; do
  echo "== $lib group $g" >> $O/ab.log
  GCMC_LIB=$PWD/paper_1408_3764_b200/$lib GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 --warps $g 2>&1 | grep -E "ctas|round ends" | tail -2 >> $O/ab.log
 done
done
