python tools/trace_lmh.py 0 > gpurun_out/trace.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
