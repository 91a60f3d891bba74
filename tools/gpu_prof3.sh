#!/bin/bash
TAG=${1:-p}
O=gpurun_out/$TAG
mkdir -p $O
GCMC_ENGINE_PROFILE=1 timeout 600 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 > $O/prof1m.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_engine -s 1 -c 1 -o $O/eng python tools/prof_engine.py --n0 1048576 --mu 1 --moves 65536 --warm 65536 > $O/ncu.log 2>&1
