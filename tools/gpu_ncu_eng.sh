#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_engine -s 1 -c 1 -o $O/eng python tools/prof_engine.py --n0 1048576 --mu 1 --moves 65536 --warm 65536 > $O/ncu.log 2>&1
