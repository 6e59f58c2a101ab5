#!/bin/bash
# Gyroid paper-scale diagnostics: memory plans and Stokes-step / steady Krylov counts per decomposition.
mkdir -p gpurun_out
timeout 900 python scripts/memplan.py gyroid 0.5:200 0.75:200 1.0:200 1.5:200 > gpurun_out/memplan_gyroid.txt 2>&1
PMNS_VERBOSE=1 timeout 600 python scripts/run_config.py gyroid max_newton=3 max_krylov=400 > gpurun_out/gyroid_hm05.txt 2>&1
PMNS_VERBOSE=1 timeout 600 python scripts/run_config.py gyroid ws_merge_h=0.75 max_newton=3 max_krylov=400 > gpurun_out/gyroid_hm075.txt 2>&1
PMNS_VERBOSE=1 timeout 900 python scripts/run_config.py gyroid ws_merge_h=1.0 max_newton=3 max_krylov=400 > gpurun_out/gyroid_hm10.txt 2>&1
