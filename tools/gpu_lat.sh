#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
GCMC_ENGINE_LATENCY=1 GCMC_ENGINE_PROFILE=1 timeout 600 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 > $O/lat.log 2>&1
