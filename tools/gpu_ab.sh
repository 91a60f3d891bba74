#!/bin/bash
# A/B on one box: engine variants (parity + speed) and energy passes.
O=gpurun_out/${1:-ab}; mkdir -p $O
for m in 1 3; do GCMC_ENERGY_MODE=$m timeout 200 python tools/time_energy.py --bf-max 262144 --sizes 32768,262144,1048576 > $O/energy_m$m.log 2>&1; done
bash tools/gpu_variants.sh ${1:-ab} 1 0 1 0
for v in 0 1; do
  GCMC_E2_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_engine_parity.py tests/test_gpu_chains.py -m gpu -q -x --timeout 600 --timeout-method=thread > $O/parity_v$v.log 2>&1
  echo "parity variant $v: $(tail -1 $O/parity_v$v.log)" >> $O/summary.txt
done
