#!/bin/bash
# Full GPU test suite and the default bench line (config 3) on the session-4 code.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/q_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_gputest.log
timeout 1500 python bench.py > gpurun_out/q_bench_cfg3.json 2> gpurun_out/q_bench_cfg3.err; echo "bench rc=$?" >> gpurun_out/q_bench_cfg3.err
timeout 600 python bench.py --config cfg4s --no-cpu-baseline > gpurun_out/q_bench_cfg4s.json 2> gpurun_out/q_bench_cfg4s.err; echo "bench rc=$?" >> gpurun_out/q_bench_cfg4s.err
