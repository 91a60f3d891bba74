#!/bin/bash
# GPU parity tests, then the engine phase profile in the bench window.
O=gpurun_out/$1; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
tail -3 $O/tests.log
GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 ${@:2} > $O/prof.log 2>&1
tail -5 $O/prof.log
