#!/bin/bash
O=gpurun_out/${1:-eab}; mkdir -p $O
timeout 300 python tools/time_energy.py --bf-max 262144 --sizes 32768,262144,1048576 > $O/energy_shift.log 2>&1
GCMC_ENERGY_RINT=1 timeout 300 python tools/time_energy.py --bf-max 262144 --sizes 32768,262144,1048576 > $O/energy_rint.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "energy" --timeout 600 > $O/energy_tests.log 2>&1
