for pool in 2 4 6 8; do
  PMNS_POOL=$pool timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pool',$pool,'ms',round(d['ms_per_step']), 'mg',round(d['solve']['t_mg_ms']), 'ml', round(d['solve']['t_ml_ms']))"
done
