#!/bin/bash
# Final session-4 records: full GPU test suite (with the half-of-config-4 transient check) and the default bench.
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/t_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gputest.log
timeout 1500 python bench.py > gpurun_out/t_bench_cfg3.json 2> gpurun_out/t_bench_cfg3.err; echo "bench rc=$?" >> gpurun_out/t_bench_cfg3.err
