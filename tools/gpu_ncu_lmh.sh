python -c "import __graft_entry__ as g; g.build()" || exit 1
TRACE_NS=${TRACE_NS:-36864} timeout 900 ncu --set full --import-source on --clock-control none -k regex:${NCU_K:-lmh_tc_kernel} --launch-skip 3 --launch-count 1 -o gpurun_out/${NCU_O:-lmh_tc_src} -f python tools/trace_lmh.py 0 > gpurun_out/ncu_lmh.log 2>&1
tail -5 gpurun_out/ncu_lmh.log
