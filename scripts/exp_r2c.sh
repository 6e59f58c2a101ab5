#!/bin/bash
L=gpurun_out/exp_r2c.log
echo "== jacobian cfg4 (role-major records)" >> $L
timeout 300 python scripts/bench_jacobian.py cfg4 40 >> $L 2>&1
echo "== trace cfg3 continuation" >> $L
PMNS_TRACE=1 PMNS_GPUTIME=1 timeout 300 python scripts/run_config.py cfg3 continuation=4 >> $L 2>&1
