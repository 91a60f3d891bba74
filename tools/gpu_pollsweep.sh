#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for ns in 0 64 256 1000; do
  echo "== poll_ns $ns" >> $O/sweep.log
  GCMC_POLL_NS=$ns GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 >> $O/sweep.log 2>&1
done
