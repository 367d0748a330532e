# ncu of the north-star call (LM head + top-k at 36,864 rows, one-list mode) and its launch list
python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
TRACE_MODES=steady TRACE_NS=36864 EVOSPEC_NOTRACE=1 ncu --set full --import-source on --clock-control none -k regex:"lmh_tc|lmh_fin64" -s 6 -c 2 -o gpurun_out/prof_lmh36k -f env NH=60 python tools/gemv_probe.py > gpurun_out/ncu_lmh36k.log 2>&1
