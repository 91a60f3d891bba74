#!/bin/bash
# Iteration check: the GPU suite, a short bench, init timing, sanitizers.
O=gpurun_out/${1:-iter}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method=thread --durations=15 > $O/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
timeout 300 python tools/time_init.py > $O/init.log 2>&1
bash tools/gpu_sanitize.sh ${1:-iter}
