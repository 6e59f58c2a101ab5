#!/bin/bash
# cfg3 (h_m = 1.0): verbose Newton / FGMRES trace of the steady Re~10 solve and of a 4-increment continuation
R=scripts/run_config.py
L=gpurun_out/exp_cfg3c.log
run() { echo "== $*" >> $L; PMNS_VERBOSE=1 timeout 420 python $R "$@" >> $L 2>&1; }
run cfg3 ws_merge_h=1.0 max_newton=8 max_krylov=300
run cfg3 ws_merge_h=1.0 continuation=4 max_newton=10 max_krylov=400
