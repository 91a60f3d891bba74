#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for cfg in "256 9" "256 11" "256 13" "256 15"; do
  set -- $cfg
  echo "== group $1 variants $2" >> $O/sweep.log
  GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 --warps $1 --variants $2 2>&1 | grep -E "ctas|round ends|sequencer" | tail -3 >> $O/sweep.log
done
