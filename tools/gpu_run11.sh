timeout 1200 python -m pytest tests -m gpu -q -x -k "ragged or batched" > gpurun_out/pytest_bt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bt.log
EVOSPEC_RAGGED_LOOP=1 timeout 1200 python -m pytest tests -m gpu -q -x -k "ragged or batched" >> gpurun_out/pytest_bt.log 2>&1; echo "pytest loop rc=$?" >> gpurun_out/pytest_bt.log
python tools/bench_bt.py > gpurun_out/bench_bt.log 2>&1
