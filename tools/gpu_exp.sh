python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for ns in 8192 16384; do TRACE_MODES=flushed,steady TRACE_NS=$ns timeout 300 python tools/trace_lmh.py > gpurun_out/trace_ks$ns.log 2>&1; done
timeout 600 python bench.py --steps 30 --warmup 5 --no-bt --no-cpu-baseline > gpurun_out/bench_ks.log 2>&1
EVOSPEC_KSPLIT=0 timeout 600 python bench.py --steps 30 --warmup 5 --no-bt --no-cpu-baseline > gpurun_out/bench_ks0.log 2>&1
