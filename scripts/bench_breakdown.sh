# cfg2 step breakdown (diagnostic; not a bench number): build / solve split per variant
for v in "${@:-PMNS_POOL=4}"; do
env $v timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; r=d['roofline']
print('$v', 'ms',round(d['ms_per_step']), 'mg',round(s['t_mg_ms']), 'ml', round(s['t_ml_ms']), 'sol', round(s['t_sol_ms']), 'kry', sum(s['krylov_iters']), 'ms/kry', round(s['t_sol_ms']/sum(s['krylov_iters']),3), 'gemvGBs', round(r['achieved']), 'mdGBs', round(r['others']['md_apply_GBps']))"
done
