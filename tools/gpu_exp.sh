python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
for c in 0 32 40 48; do EVOSPEC_COMPACT_AT=$c TRACE_MODES=steady TRACE_NS=36864 timeout 300 python tools/trace_lmh.py > gpurun_out/trace_c$c.log 2>&1; done
