for v in tma v1 tma v1; do echo "scan=$v"; EVOSPEC_SCAN=$v timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-bt --steps 20 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(l['value'], {k:round(v['us'],1) for k,v in l['breakdown'].items()})"; done > gpurun_out/scanpf.log 2>&1
