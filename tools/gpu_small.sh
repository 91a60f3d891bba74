#!/bin/bash
# Small-N engine shapes: engine2 at several CTA counts vs the per-window engine.
O=gpurun_out/$1; mkdir -p $O; : > $O/small.log
for n0mu in "2048 -2" "2048 1" "32768 1"; do
  set -- $n0mu
  for c in 0 10 17 33 65; do
    echo "== n0 $1 mu $2 engine2 ctas $c" >> $O/small.log
    timeout 120 python tools/prof_engine.py --n0 $1 --mu $2 --moves 1048576 --warm 1048576 --ctas $c 2>&1 | grep -E "ctas=|rror" | tail -2 >> $O/small.log
  done
  for c in 0 9 33; do
    echo "== n0 $1 mu $2 per-window engine ctas $c" >> $O/small.log
    GCMC_ENGINE_V1=1 timeout 120 python tools/prof_engine.py --n0 $1 --mu $2 --moves 1048576 --warm 1048576 --ctas $c 2>&1 | grep -E "ctas=|rror" | tail -2 >> $O/small.log
  done
done
cat $O/small.log
