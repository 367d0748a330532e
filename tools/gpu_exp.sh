# scratch experiment: split-K of the two-list head's dynamic tiles
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "draft or two_list or oov or sharded" > gpurun_out/exp_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/exp_pytest.log
tail -3 gpurun_out/exp_pytest.log
for P in 1 4 2 1 4 2; do
  echo "P=$P"; EVOSPEC_DYN_SPLIT=$P timeout 300 python bench.py --no-bt --no-extra --no-sweep --no-cpu --steps 200 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d['value'])"
done
for P in 1 4; do EVOSPEC_DYN_SPLIT=$P timeout 300 python tools/trace_step.py > gpurun_out/exp_trace_P$P.log 2>&1; tail -25 gpurun_out/exp_trace_P$P.log; done
