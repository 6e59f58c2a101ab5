# nested-dissection leaf-size sweep on cfg2 (diagnostic; not a bench number)
for leaf in 128 256 512; do
PMNS_ND_LEAF=$leaf timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; r=d['roofline']
print('leaf=$leaf', 'ms',round(d['ms_per_step']), 'mg',round(s['t_mg_ms']), 'ml', round(s['t_ml_ms']), 'sol', round(s['t_sol_ms']), 'ms/kry', round(s['t_sol_ms']/sum(s['krylov_iters']),3), 'mpGB', round(s['stored_bytes']['mp_bytes']/1e9,2), 'gemvGBs', round(r['achieved']))"
done
PMNS_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "pmns nd\]|timeline|pmns build\] [A-Za-z]" | tail -40
