python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/trace_step.py > gpurun_out/trace_step.log 2>&1
for i in 1 2; do timeout 600 python bench.py --steps 100 --warmup 5 --no-bt --no-sweep --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step_us', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['value']), 'flags', d['device_flags'])"; done > gpurun_out/bench_quick.log 2>&1
