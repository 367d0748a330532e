for st in 3 4 5 6; do echo "stages<=$st"; EVOSPEC_STAGES=$st python tools/trace_lmh.py 0 2>&1 | grep -E "median|prod_done|end  "; done > gpurun_out/stages.log 2>&1
