for rs in 8 4 2; do for fp in 0 1; do echo "rs=$rs fp32test=$fp"; if [ $fp = 1 ]; then export EVOSPEC_SCAN_FP32TEST=1; else unset EVOSPEC_SCAN_FP32TEST; fi; EVOSPEC_SCAN_RS=$rs timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-bt --no-extra --steps 20 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(l['value'], {k:round(v['us'],1) for k,v in l['breakdown'].items()})"; done; done > gpurun_out/fp32test.log 2>&1
