timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not cfg2" 2>&1 | tail -1
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run',$rep,'ms',round(d['ms_per_step']), 'mg',round(d['solve']['t_mg_ms']), 'ml', round(d['solve']['t_ml_ms']), 'sol', round(d['solve']['t_sol_ms']), 'frac', round(d['roofline']['frac'],3))"
done
