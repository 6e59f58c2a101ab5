#!/bin/bash
# Round 2 (session 4) experiments: config-4 memory plans per decomposition, a traced config-3 build, the DMMA
# GEMM's rates, and a full ncu capture of the J apply at config-4 size.
mkdir -p gpurun_out
timeout 600 python scripts/dgemm_rates.py > gpurun_out/dgemm_rates.txt 2>&1
timeout 900 python scripts/trace_build.py cfg3 1 > gpurun_out/trace_build_cfg3.txt 2>&1
timeout 900 python scripts/bench_jacobian.py cfg4 20 > gpurun_out/jbench_cfg4.json 2> gpurun_out/jbench_cfg4.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:apply_kernel -c 1 \
   -o gpurun_out/r02_japply_cfg4 python scripts/bench_jacobian.py cfg4 2 > gpurun_out/ncu_japply.log 2>&1
timeout 2400 python scripts/memplan.py cfg4 0.5:50 0.25:50 0:50 0:25 0.5:200 > gpurun_out/memplan_cfg4.txt 2>&1
