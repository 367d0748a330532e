# finalisation A/B: parity suite on the new finalisation, then traces (new vs fin32)
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K} > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
TRACE_MODES=flushed,steady TRACE_NS=36864 timeout 300 python tools/trace_lmh.py > gpurun_out/trace_fin64.log 2>&1
TRACE_MODES=steady TRACE_NS=8192 timeout 300 python tools/trace_lmh.py > gpurun_out/trace_fin64_8192.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 5 --no-bt --no-extra --no-cpu-baseline > gpurun_out/bench_fin64.log 2>&1
