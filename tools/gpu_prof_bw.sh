#!/bin/bash
# Engine phase profile in the bench window (1M, mu=+1, moves 12.6M..16.8M).
O=gpurun_out/$1; mkdir -p $O
GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 ${@:2} > $O/prof.log 2>&1
tail -6 $O/prof.log
