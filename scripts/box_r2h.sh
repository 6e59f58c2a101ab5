#!/bin/bash
# Round 2 (session 4) first box call: full GPU test suite and the default bench line (config 3, roofline on the
# oracle's SuperLU nnz, all-cores oracle baseline).
mkdir -p gpurun_out
( nproc; free -g; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,memory.total --format=csv ) > gpurun_out/host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 1200 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
echo "bench rc=$?" >> gpurun_out/bench_cfg3.err
