#!/bin/bash
# A/B of GCMC_E2_VARIANT values at 1M (prof_engine) and on the 64k sweep (K=6), plus parity for the variant.
O=gpurun_out/${1:-ab2}; mkdir -p $O; shift
for v in "$@"; do
  GCMC_E2_VARIANT=$v timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 > $O/v$v.log 2>&1
  echo "1M variant $v: $(tail -1 $O/v$v.log)" >> $O/summary.txt
  GCMC_E2_VARIANT=$v timeout 600 python bench.py --sweep --chains-per-gpu 6 --steps 3 --warmup 3 --no-cpu-baseline --no-energy > $O/sweep_v$v.log 2>&1
  python -c "
import json; l=json.loads(open('$O/sweep_v$v.log').read().strip().splitlines()[-1])
print('sweep K=6 variant $v', 'value %.4g'%l['value'], 'mpr %.1f'%l['moves_per_round'], 'nspr %.0f'%l['ns_per_round'])" >> $O/summary.txt
done
GCMC_E2_VARIANT=${!#} timeout 900 python -m pytest tests/test_gpu_engine_parity.py tests/test_gpu_chains.py -m gpu -q --timeout 600 > $O/parity.log 2>&1
tail -1 $O/parity.log >> $O/summary.txt
