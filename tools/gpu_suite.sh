O=gpurun_out/r02d
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' > $O/lscpu.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > $O/gpu_tests.log 2>&1
echo "pytest rc=$?" >> $O/gpu_tests.log
#timeout 600 python bench.py > $O/bench.log 2>&1
echo done
