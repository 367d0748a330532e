python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
for v in "60 8" "60 5" "60 4" "16 8" "16 6" "32 8"; do set -- $v
  EVOSPEC_TC_SMAX=$2 TRACE_NH=$1 TRACE_MODES=steady TRACE_NS=36864 timeout 300 python tools/trace_lmh.py > gpurun_out/trace_nh$1_s$2.log 2>&1
done
