#!/bin/bash
# Iteration check: energy timing, the GPU suite, a short bench.
O=gpurun_out/${1:-iter}; mkdir -p $O
timeout 300 python tools/time_energy.py --bf-max 262144 --sizes 32768,262144,1048576 > $O/energy.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method=thread --durations=15 > $O/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
