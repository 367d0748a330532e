python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_kd.py tests/test_gpu_parity.py -q -k "sharded or kd or invariant or envelope or hl_kernel or llama_full" > gpurun_out/pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu2.log
