#!/bin/bash
# cfg3: full steady Re~10 solves (Stokes step + gPLMM Newton) vs watershed merge threshold h_m
R=scripts/run_config.py
L=gpurun_out/exp_cfg3b.log
run() { echo "== $*" >> $L; timeout 400 python $R "$@" >> $L 2>&1; }
run cfg3 ws_merge_h=1.0
run cfg3 ws_merge_h=0.75 max_newton=1
run cfg3 ws_merge_h=1.5 max_newton=1
run cfg3 ws_merge_h=1.0 continuation=2
run cfg2 ws_merge_h=1.0
