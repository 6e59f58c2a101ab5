#!/bin/bash
# Long box call: the config-3 oracle goldens need more host memory (>60 GB) than the build container has, so they run
# on the GPU box's host in the background while the GPU runs the test suite, config 3s and a bench line.
mkdir -p gpurun_out/golden
cp tests/golden/cfg3_stokes.json gpurun_out/golden/old_cfg3_stokes.json 2>/dev/null
( timeout 6600 python scripts/oracle_golden.py cfg3 stokes nnz > gpurun_out/golden/cfg3_golden.log 2>&1; \
  cp tests/golden/cfg3_stokes.json tests/golden/cfg3_factor_nnz.json gpurun_out/golden/ 2>/dev/null ) &
OPID=$!
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest4.log 2>&1
PMNS_VERBOSE=1 timeout 600 python scripts/run_config.py cfg3s continuation=4 2>&1 | grep -v "fgmres\|pmns nd\|gputime" > gpurun_out/cfg3s_gpu.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_cfg3_b.json 2> gpurun_out/bench_cfg3_b.err
wait $OPID
free -g >> gpurun_out/golden/cfg3_golden.log
