# scratch experiment: early dynamic list + last static tile folded as the last tile
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "two_list or draft_step or ragged" > gpurun_out/exp_pytest0.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_pytest0.log
tail -3 gpurun_out/exp_pytest0.log
grep -q "rc=0" gpurun_out/exp_pytest0.log || exit 1
for E in 1 0 1 0; do echo "EARLY=$E"; EVOSPEC_EARLY_LIST=$E timeout 300 python bench.py --no-bt --no-extra --no-sweep --no-cpu --steps 200 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['value'], d['e2e']['value'])"; done
timeout 300 python tools/trace_step.py > gpurun_out/exp_trace.log 2>&1; sed -n 1,16p gpurun_out/exp_trace.log; grep -A9 "lmh start" gpurun_out/exp_trace.log | tail -10
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/exp_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_pytest.log
tail -3 gpurun_out/exp_pytest.log
