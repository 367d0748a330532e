for g in 0 1; do echo "nograph=$g"; if [ $g = 1 ]; then export EVOSPEC_NO_GRAPH=1; else unset EVOSPEC_NO_GRAPH; fi; timeout 600 python bench.py --no-cpu-baseline --no-sweep --no-bt --no-extra --steps 30 2>&1 | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print(l['value'], l['ms_per_step'], l['e2e']['value'], l['gpu_launches'])"; done > gpurun_out/graph.log 2>&1
