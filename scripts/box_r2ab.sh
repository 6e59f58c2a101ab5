#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/dgemm_rates.py > gpurun_out/ab_dgemm_rates.txt 2>&1
timeout 600 python scripts/trace_build.py cfg3 2 > gpurun_out/ab_trace_build_cfg3.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/ab_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/ab_kernels.log
