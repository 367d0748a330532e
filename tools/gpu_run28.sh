for nc in 0 1; do echo "nocompute=$nc"; if [ $nc = 1 ]; then export EVOSPEC_SCAN_NOCOMPUTE=1; else unset EVOSPEC_SCAN_NOCOMPUTE; fi; timeout 600 python bench.py --steps 20 --no-cpu-baseline --no-sweep --no-bt --no-extra 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(l['value'], {k:round(v['us'],1) for k,v in l['breakdown'].items()})"; done > gpurun_out/nocompute.log 2>&1
