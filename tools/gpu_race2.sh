python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 99 python -m pytest tests -m gpu -q -x -k "odd_shapes or test_kd_loss or coverage or subset_update and random or multitile and 10-False" > gpurun_out/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_racecheck.log
tail -3 gpurun_out/sanitizer_racecheck.log
timeout 600 python -m pytest tests/test_gpu_coverage.py -m gpu -q 2>&1 | tail -1
AB_VARIANTS="new" bash tools/gpu_ab.sh
timeout 300 python bench.py --steps 10 --no-sweep --no-bt --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('coverage us', l['extra_configs']['coverage']['us'], l['extra_configs']['coverage']['mean_recall'])"
