#!/bin/bash
# Records: config-2 bench line (continuity with round 1) and a full ncu capture of the build's dominant kernel
# (grouped fp64 DMMA GEMM) at config 3.
mkdir -p gpurun_out
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/aa_bench_cfg2.json 2> gpurun_out/aa_bench_cfg2.err; echo "rc=$?" >> gpurun_out/aa_bench_cfg2.err
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dgemm_grouped -s 30 -c 1 \
   -o gpurun_out/r02_dgemm_grouped_cfg3 python scripts/trace_build.py cfg3 0 > gpurun_out/aa_ncu_dgemm.log 2>&1
