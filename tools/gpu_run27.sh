for i in 1 2; do timeout 600 python bench.py --steps 30 --no-cpu-baseline --no-sweep --no-bt --no-extra 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(l['value'], {k:round(v['us'],1) for k,v in l['breakdown'].items()})"; done > gpurun_out/scan2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
