python tools/trace_build.py > gpurun_out/trace_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-bt --no-extra --steps 30 > gpurun_out/bench.log 2>&1
