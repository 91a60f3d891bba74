#!/bin/bash
# Chain-per-SM engine: parity tests, role cycles (GCMC_SM_PHASES), K=148 sweep rate.
mkdir -p gpurun_out/${1:-sm}
O=gpurun_out/${1:-sm}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engine_sm.py -x -q > $O/tests.log 2>&1
tail -2 $O/tests.log
GCMC_SM_PHASES=1 timeout 300 python tools/sm_sweep.py --mode 2 --k 1 --reps 1 > $O/phases.jsonl 2> $O/phases.err
tail -2 $O/phases.err; cat $O/phases.jsonl
timeout 600 python tools/sm_sweep.py --mode 2 --k ${KS:-148} > $O/sweep.jsonl 2> $O/sweep.err; cat $O/sweep.jsonl; tail -2 $O/sweep.err
