TRACE_NS=8192,36864 timeout 120 python tools/trace_hl.py > gpurun_out/trace_hl.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "integer or tiny or medium or duplicate or empty or lmh_paths or multitile or tc_integer or llama_full" > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
