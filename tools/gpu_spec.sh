#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
GCMC_SPEC=1 GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 > $O/spec1.log 2>&1
GCMC_SPEC=0 GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 > $O/spec0.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
