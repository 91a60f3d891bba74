#!/bin/bash
# quick engine2 check: smoke, selected parity tests, short bench
O=gpurun_out/${1:-q}
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "${2:-first_1e5_moves_identical or maintained or chunk or per_window}" > $O/tests.log 2>&1
GCMC_ENGINE_PROFILE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/bench.log 2>&1
echo done
