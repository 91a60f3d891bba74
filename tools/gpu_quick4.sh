#!/bin/bash
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
GCMC_ENGINE_PROFILE=1 timeout 600 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 > $O/prof1m.log 2>&1
GCMC_ENGINE_PROFILE=1 timeout 600 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 --warps 256 > $O/prof1m_256.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
echo "tests rc=$?" >> $O/gpu_tests.log
