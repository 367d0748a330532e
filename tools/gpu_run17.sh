for lt in 128 32; do echo "last_tile=$lt"; EVOSPEC_LAST_TILE=$lt python tools/trace_lmh.py 0 2>&1 | grep -E "median|prod_done|t0_|t1_|end|fin_end|ncand"; done > gpurun_out/lasttile.log 2>&1
TRACE_NS=8192 python tools/trace_lmh.py 0 2>&1 | grep -E "median|prod_done|t0_|end|fin_end|ncand" >> gpurun_out/lasttile.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
