# A/B: the committed tree (_head worktree) vs the working tree, bench sweep only
python -c "import __graft_entry__ as g; g.build()" || exit 1
run() { timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-bt --no-extra 2>/dev/null | tail -1 | python -c "
import json,sys
l=json.loads(sys.stdin.read()); print('$1', round(l['value']), {k:round(v['us'],1) for k,v in l['breakdown'].items()}, [(r['n_S'], round(r['us'],1), round(r.get('us_steady',0),1)) for r in l['subset_sweep']])"; }
for v in ${AB_VARIANTS:-new head par0}; do
  case $v in
    new) run new ;;
    par0) EVOSPEC_PAR_FOLD=0 run par0 ;;
    head) (cd _head && run head) ;;
    headB) (cd _headB && run headB) ;;
    headC) (cd _headC && run headC) ;;
    fin*) EVOSPEC_FIN_OPT=${v#fin} run $v ;;
    nt512) EVOSPEC_FIN_NT=512 run nt512 ;;
  esac
done
