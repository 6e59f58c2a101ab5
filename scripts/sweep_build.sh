# Build-plan cost-model sweep on cfg2 (diagnostic; not a bench number)
run() {
  env "$@" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print('$*','ms',round(d['ms_per_step']), 'mg',round(s['t_mg_ms']), 'ml', round(s['t_ml_ms']), 'sol', round(s['t_sol_ms']), 'kry', sum(s['krylov_iters']), 'mpGB', round(s['stored_bytes']['mp_bytes']/1e9,2))"
}
run PMNS_COST_GFLOPS=10000
run PMNS_COST_GFLOPS=20000
run PMNS_COST_GFLOPS=40000
run PMNS_COST_GFLOPS=20000 PMNS_COST_APPLY_PCT=50
run PMNS_COST_GFLOPS=20000 PMNS_COST_APPLY_PCT=200
run PMNS_POOL=6
