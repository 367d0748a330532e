# LM-head phase trace in three modes (flushed / code warmed / steady) at 36,864 and 8,192 rows
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
for ns in 36864 8192; do TRACE_NS=$ns timeout 300 python tools/trace_lmh.py > gpurun_out/trace_lmh_$ns.log 2>&1; done
timeout 600 python bench.py --steps 50 --warmup 5 --no-bt --no-extra --no-cpu-baseline > gpurun_out/bench_base.log 2>&1
