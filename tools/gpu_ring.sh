python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_scan_ring.py tests/test_abi.py -q > gpurun_out/ring_test.log 2>&1; echo "rc=$?" >> gpurun_out/ring_test.log
