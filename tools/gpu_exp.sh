# experiment runner: build, the scan/union parity subset, Bt breakdown, one bench line
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_scan_ring.py tests/test_gpu_parity.py -q -x -k "scan_ring or llama_full or union_selection or medium" > gpurun_out/exp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/exp_tests.log
timeout 300 python tools/trace_bt.py > gpurun_out/trace_bt.log 2>&1
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_exp.log 2>&1
