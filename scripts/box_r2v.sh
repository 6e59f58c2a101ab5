#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_loopback.py tests/test_gpu_parity.py -m "gpu and not slow" -q -x -k "loopback or partition or nccl or memory_plan" > gpurun_out/v_disttest.log 2>&1; echo "rc=$?" >> gpurun_out/v_disttest.log
