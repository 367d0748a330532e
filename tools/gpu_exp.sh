python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
TRACE_MODES=steady TRACE_NS=36864 timeout 300 python tools/trace_lmh.py > gpurun_out/trace_rows.log 2>&1
