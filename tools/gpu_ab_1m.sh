#!/bin/bash
# engine2 round-size A/B at 1M (library variants built with tools/build_variant.py NAME -DGCMC_E2_MOVES=M).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
L=$PWD/paper_1408_3764_b200
timeout 300 python tools/ab_1m.py 2>&1 | tail -1
for v in $VARIANTS; do GCMC_LIB=$L/libgcmc_b200_$v.so timeout 300 python tools/ab_1m.py 2>&1 | tail -1; done
