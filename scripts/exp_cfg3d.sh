#!/bin/bash
# Krylov stagnation in later Newton steps: composition with J^k (A18) vs the build-time J(x_b); restart size
R=scripts/run_config.py
L=gpurun_out/exp_cfg3d.log
run_c() { echo "== COMPOSE=1 $*" >> $L; PMNS_COMPOSE=1 timeout 300 python $R "$@" >> $L 2>&1; }
run() { echo "== $*" >> $L; timeout 300 python $R "$@" >> $L 2>&1; }
run_c cfg3 ws_merge_h=1.0 continuation=4 max_newton=10 max_krylov=400
run cfg3 ws_merge_h=1.0 continuation=4 max_newton=10 max_krylov=600 restart=150
run cfg2 p_in=2977 max_krylov=400 max_newton=12
run_c cfg2 p_in=2977 max_krylov=400 max_newton=12
run cfg2 p_in=2977 max_krylov=400 max_newton=12 continuation=4
