python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:union_kernel -s 3 -c 1 -o gpurun_out/prof_union -f python tools/trace_build.py > gpurun_out/ncu_union.log 2>&1
