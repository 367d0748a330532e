set -x
python tools/trace_lmh.py 0 > gpurun_out/trace.log 2>&1
python tools/trace_build.py > gpurun_out/trace_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lmh_tc" -s 2 -c 1 -o gpurun_out/prof6 python tools/trace_lmh.py 0 > gpurun_out/ncu6.log 2>&1
