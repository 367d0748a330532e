# build, GPU parity suite, LM-head trace (iteration helper)
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -z "$SKIP_TESTS" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log; fi
bash tools/gpu_trace.sh
if [ -n "$ALSO_OLD" ]; then EVOSPEC_PAR_FOLD=0 bash tools/gpu_trace.sh; fi
