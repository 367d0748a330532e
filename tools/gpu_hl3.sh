for e in 0 512; do echo "== EXP=$e"; EVOSPEC_HL_EXP=$e TRACE_NS=8192,36864 timeout 120 python tools/trace_hl.py 2>&1 | grep -E "n_S=|t0_ready|stored|clock64"; done > gpurun_out/trace_exp.log
