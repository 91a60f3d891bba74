#!/bin/bash
# 64k mu sweep with K chains per GPU (bench.py --sweep --chains-per-gpu K), then the chain / engine parity tests.
O=gpurun_out/${1:-sweep}; mkdir -p $O; shift
for K in "$@"; do
  timeout 900 python bench.py --sweep --chains-per-gpu $K --steps 3 --warmup 3 > $O/sweep_k$K.log 2>&1
  python -c "
import json; l=json.loads(open('$O/sweep_k$K.log').read().strip().splitlines()[-1])
print('K=$K', 'value %.4g'%l['value'], 'mpr %.1f'%l['moves_per_round'], 'nspr %.0f'%l['ns_per_round'], 'cpu', (l.get('cpu_baseline') or {}).get('value'), 'same', (l.get('cpu_gpu_same_trajectory') or {}).get('all'))" >> $O/summary.txt
done
timeout 900 python -m pytest tests/test_gpu_chains.py tests/test_gpu_engine_parity.py -m gpu -q --timeout 600 > $O/parity.log 2>&1
tail -1 $O/parity.log >> $O/summary.txt
