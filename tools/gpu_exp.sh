python -c "import paper_2605_27390_b200._build as b; b.build()" > gpurun_out/build.log 2>&1
for v in 0 1; do for ns in 8192 16384; do EVOSPEC_PAR_SINGLE=$v TRACE_MODES=flushed,steady TRACE_NS=$ns timeout 300 python tools/trace_lmh.py > gpurun_out/trace_ps${v}_$ns.log 2>&1; done; done
EVOSPEC_PAR_SINGLE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or medium or lmh_paths or integer or ties or odd or empty or duplicate" > gpurun_out/pytest_ps.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ps.log
