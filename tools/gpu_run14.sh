timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-bt > gpurun_out/bench.log 2>&1
EVOSPEC_SCAN=v1 timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-bt > gpurun_out/bench_v1.log 2>&1
