python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "draft_step" 2>&1 | tail -2
for pf in 1 0 1 0; do EVOSPEC_DYN_PF=$pf timeout 600 python bench.py --steps 50 --no-sweep --no-bt --no-extra --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; l=json.loads(sys.stdin.read()); print('dyn_pf=$pf', round(l['value']), round(l['ms_per_step']*1e3,1), 'e2e', round(l['e2e']['value']))"; done
