python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
TRACE_MODES=flushed,steady TRACE_NS=36864 timeout 300 python tools/trace_lmh.py > gpurun_out/trace_w.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-bt --no-extra --no-cpu-baseline > gpurun_out/bench_w.log 2>&1
