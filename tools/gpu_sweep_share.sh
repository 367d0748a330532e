python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
for sh in 16 12 8 6 4; do
  echo "== EVOSPEC_DYN_SHARE=$sh"
  EVOSPEC_DYN_SHARE=$sh timeout 300 python tools/trace_step.py | grep -E "union end|lmh (prod_done|end)|fin end"
  EVOSPEC_DYN_SHARE=$sh timeout 300 python bench.py --steps 100 --warmup 5 --no-bt --no-sweep --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_us', round(d['ms_per_step']*1e3,1))"
done > gpurun_out/sweep_share.log 2>&1
