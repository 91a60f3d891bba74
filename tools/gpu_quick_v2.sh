#!/bin/bash
# quick engine2 check: smoke, selected parity tests, short bench
O=gpurun_out/${1:-q}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
if [ -n "$2" ]; then K="-k $2"; else K=""; fi; timeout 900 python -m pytest tests -m gpu -x -q $K > $O/tests.log 2>&1
GCMC_ENGINE_PROFILE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
echo done
