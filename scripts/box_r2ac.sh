#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --deselect tests/test_gpu_parity.py::test_cfg2_end_to_end > gpurun_out/ac_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/ac_gputest.log
timeout 600 python scripts/trace_build.py cfg3 2 > gpurun_out/ac_trace_build_cfg3.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ac_bench_cfg3.json 2> gpurun_out/ac_bench_cfg3.err; echo "rc=$?" >> gpurun_out/ac_bench_cfg3.err
