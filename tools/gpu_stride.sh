python -c "import __graft_entry__ as g; g.build()" || exit 1
for st in 1 4 37 1 4 37; do EVOSPEC_DYN_STRIDE=$st timeout 600 python bench.py --steps 50 --no-sweep --no-bt --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('stride=$st', round(l['value']), round(l['ms_per_step']*1e3,1))"; done
