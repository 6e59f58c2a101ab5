#!/bin/bash
L=gpurun_out/exp_r2f.log
for n in 2 3; do
  echo "== cfg3 continuation=$n" >> $L
  timeout 400 python scripts/run_config.py cfg3 continuation=$n >> $L 2>&1
done
echo "== cfg3 trace (warm builds)" >> $L
PMNS_TRACE=1 PMNS_VERBOSE=1 timeout 300 python scripts/run_config.py cfg3 continuation=4 2>&1 | grep "pmns nd\] M_p+Abar level\|nd_factor\|allocator\|concurrent" | tail -30 >> $L
