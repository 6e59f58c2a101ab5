#!/bin/bash
mkdir -p gpurun_out
PMNS_VERBOSE=1 timeout 1500 python scripts/run_transient_check.py cfg4h > gpurun_out/s_cfg4h.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --deselect tests/test_gpu_parity.py::test_cfg2_end_to_end > gpurun_out/s_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/s_gputest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s_bench_cfg3.json 2> gpurun_out/s_bench_cfg3.err; echo "rc=$?" >> gpurun_out/s_bench_cfg3.err
