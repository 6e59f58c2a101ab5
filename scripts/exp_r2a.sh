#!/bin/bash
# after the A18 revision (composition with J(x_b)): cfg3 (h_m = 1.0) steady and continuation; J-apply bandwidth at cfg4 size
R=scripts/run_config.py
L=gpurun_out/exp_r2a.log
run() { echo "== $*" >> $L; PMNS_VERBOSE=1 timeout 300 python $R "$@" 2>&1 | grep -v fgmres >> $L; }
run cfg3 ws_merge_h=1.0 max_newton=30 max_krylov=600
run cfg3 ws_merge_h=1.0 continuation=4
echo "== jacobian cfg4" >> $L
timeout 300 python scripts/bench_jacobian.py cfg4 40 >> $L 2>&1
