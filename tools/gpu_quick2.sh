#!/bin/bash
# quick engine check on the GPU box: parity suite + 1M throughput
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1
echo "tests rc=$?" >> $O/gpu_tests.log
timeout 600 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 > $O/prof1m.log 2>&1
timeout 300 python tools/prof_engine.py --n0 32768 --mu -2 --moves 262144 --warm 100000 > $O/prof32k.log 2>&1
