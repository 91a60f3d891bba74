#!/bin/bash
# 64k mu-sweep with many chains per GPU (chain-per-SM engine): bench lines and tests.
mkdir -p gpurun_out/${1:-swsm}
O=gpurun_out/${1:-swsm}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_engine_sm.py tests/test_gpu_chains.py -x -q > $O/tests.log 2>&1
tail -2 $O/tests.log
lscpu | grep -E "Model name|^CPU\(s\)" > $O/lscpu.txt; cat $O/lscpu.txt
for K in ${KS:-128 148}; do
  timeout 900 python bench.py --sweep --chains-per-gpu $K --steps 3 --warmup 3 --no-energy > $O/bench_k$K.json 2> $O/bench_k$K.err
  python - $O/bench_k$K.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(d["config"]["chains"], "value %.4g e2e %.4g"%(d["value"], d["e2e"]["value"]), "cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["cores"], "engine", d.get("engine"), "same", (d.get("cpu_gpu_same_trajectory") or {}).get("all"), "mpr %.1f nsr %.0f"%(d["moves_per_round"], d["ns_per_round"]), d["clocks"])
PY
  tail -2 $O/bench_k$K.err
done
