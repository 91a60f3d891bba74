#!/bin/bash
# Engine parity tests under several GCMC_E2_VARIANT values (A/B correctness).
O=gpurun_out/${1:-pv}; mkdir -p $O; shift
for v in "$@"; do
  GCMC_E2_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_engine_parity.py tests/test_gpu_chains.py -m gpu -q -x --timeout 600 --timeout-method=thread > $O/parity_v$v.log 2>&1
  echo "variant $v: $(tail -1 $O/parity_v$v.log)" >> $O/summary.txt
done
