#!/bin/bash
# Session 4: large-tile GEMM + warp-per-row extend-add: kernel tests, parity tests (without the slow full-size ones),
# GEMM rates, a traced config-3 build and the config-3 bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/k_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/k_kernels.log
timeout 300 python scripts/dgemm_rates.py > gpurun_out/k_dgemm_rates.txt 2>&1
timeout 600 python scripts/trace_build.py cfg3 1 > gpurun_out/k_trace_build_cfg3.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --deselect tests/test_gpu_parity.py::test_cfg2_end_to_end > gpurun_out/k_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/k_gputest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/k_bench_cfg3.json 2> gpurun_out/k_bench_cfg3.err; echo "rc=$?" >> gpurun_out/k_bench_cfg3.err
PMNS_VERBOSE=1 timeout 900 python scripts/run_config.py gyroid ws_merge_h=0.75 max_newton=8 max_krylov=600 > gpurun_out/k_gyroid_hm075.txt 2>&1
