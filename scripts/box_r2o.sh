#!/bin/bash
# U buckets by (child level, parent level), panel-width dispatch of the multi-RHS solves, M_d after M_p on big
# problems: parity tests, traced config-3 build, config-4h transient, config-3 bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --deselect tests/test_gpu_parity.py::test_cfg2_end_to_end > gpurun_out/o_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/o_gputest.log
timeout 600 python scripts/trace_build.py cfg3 2 > gpurun_out/o_trace_build_cfg3.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/o_bench_cfg3.json 2> gpurun_out/o_bench_cfg3.err; echo "rc=$?" >> gpurun_out/o_bench_cfg3.err
PMNS_VERBOSE=1 timeout 2400 python scripts/run_transient_check.py cfg4h > gpurun_out/o_cfg4h.txt 2>&1
