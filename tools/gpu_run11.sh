timeout 1200 python -m pytest tests -m gpu -q -x -k "ragged or batched" > gpurun_out/pytest_bt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bt.log
