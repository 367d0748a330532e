for wn in 0 1; do echo "w_normal=$wn"; if [ $wn = 1 ]; then export EVOSPEC_W_NORMAL=1; else unset EVOSPEC_W_NORMAL; fi; python tools/trace_lmh.py 0 2>&1 | grep -E "median|fin_end|clock64"; timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-bt --no-extra 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(l['value'], [(r['n_S'], round(r['us'],1), r.get('us_steady')) for r in l['subset_sweep']])"; done > gpurun_out/wpol.log 2>&1
