python -c "import __graft_entry__ as g; g.build()" || exit 1
rm -f gpurun_out/trace_lmh.log
for ns in ${TRACE_SIZES:-36864 8192}; do TRACE_NS=$ns timeout 300 python tools/trace_lmh.py 0 >> gpurun_out/trace_lmh.log 2>&1; done
cat gpurun_out/trace_lmh.log
