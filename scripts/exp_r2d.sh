#!/bin/bash
L=gpurun_out/exp_r2d.log
timeout 900 python -m pytest tests/test_dist_loopback.py -x -q > gpurun_out/loopback.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse_colour or cell_records" >> gpurun_out/loopback.log 2>&1
echo "== trace cfg3 continuation (warm builds)" >> $L
PMNS_TRACE=1 PMNS_VERBOSE=1 timeout 300 python scripts/run_config.py cfg3 continuation=4 2>&1 | grep -v "fgmres\|newton\]" >> $L
