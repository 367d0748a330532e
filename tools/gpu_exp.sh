python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_scan_ring.py tests/test_gpu_parity.py -x -q -k "scan_ring or llama_full or union_selection or medium or tiny or draft" > gpurun_out/pytest_scan.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_scan.log
for i in 1 2; do timeout 600 python bench.py --steps 50 --warmup 5 --no-bt --no-extra --no-cpu-baseline --no-sweep > gpurun_out/bench_s$i.log 2>&1; done
timeout 300 python tools/trace_step.py > gpurun_out/trace_step.log 2>&1
