python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_oov.py -q -x > gpurun_out/union_tests.log 2>&1; echo "rc=$?" >> gpurun_out/union_tests.log
timeout 300 python tools/trace_build.py > gpurun_out/trace_union.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_union.log 2>&1
