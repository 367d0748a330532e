python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
python tools/gemv_probe.py > gpurun_out/gemv_probe.log 2>&1
NH=4 python tools/gemv_probe.py >> gpurun_out/gemv_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gemv or lmh_paths or tiny or medium" > gpurun_out/pytest_gemv.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gemv.log
