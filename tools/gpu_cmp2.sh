timeout 600 python bench.py --no-cpu-baseline --no-bt --no-extra --steps 30 2>&1 | tail -1 | python3 -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',round(d['value']),'ms',round(d['ms_per_step'],4),'e2e',round(d['e2e']['value']))
print('breakdown',{k:round(v['us'],1) for k,v in d['breakdown'].items()})
print('sweep',[(r['n_S'],round(r['us'],1),round(r.get('us_steady',0),1)) for r in d['subset_sweep']])
print('per_depth', d['per_depth'])
" > gpurun_out/cmp2.log 2>&1
