#!/bin/bash
# cfg3 convergence diagnosis: Stokes-step Krylov counts under drive / decomposition / restart variants
# (scripts/run_config.py; max_newton=1 = the Stokes step only).  Output: gpurun_out/exp_cfg3.log
R=scripts/run_config.py
L=gpurun_out/exp_cfg3.log
run() { echo "== $*" >> $L; timeout 300 python $R "$@" >> $L 2>&1; }
run cfg3 max_newton=1
run cfg3 max_newton=1 body_force=0,0,0 p_in=3234
run cfg2 max_newton=1 body_force=458,0,0 p_in=0
run cfg2 max_newton=1
run cfg3 max_newton=1 ws_merge_h=1.0
run cfg3 max_newton=1 ws_merge_h=2.0
run cfg3 max_newton=1 ws_min_cells=200
run cfg3 max_newton=1 dual_layers=2
