#!/bin/bash
L=gpurun_out/exp_r2e.log
free -g > gpurun_out/box_info.txt; nproc >> gpurun_out/box_info.txt
timeout 900 python -m pytest tests/test_dist_loopback.py -x -q > gpurun_out/loopback.log 2>&1
echo "== trace cfg3 continuation (allocator eviction)" >> $L
PMNS_TRACE=1 PMNS_VERBOSE=1 timeout 300 python scripts/run_config.py cfg3 continuation=4 2>&1 | grep "allocator\|concurrent\|dual thread\|nd_factor\|^{" >> $L
echo "== cfg4 transient 2 steps" >> $L
PMNS_VERBOSE=1 timeout 600 python scripts/run_config.py cfg4 transient=2 max_krylov=300 2>&1 | grep -v "fgmres\|pmns nd\]\|gputime" | tail -40 >> $L
