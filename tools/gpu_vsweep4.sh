#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for cfg in "256 11" "128 11" "128 13" "128 15"; do
  set -- $cfg
  echo "== group $1 variants $2" >> $O/sweep.log
  GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 --warps $1 --variants $2 2>&1 | grep -E "ctas|round ends|sequencer|evaluator" | tail -4 >> $O/sweep.log
done
