#!/bin/bash
# config-3 oracle goldens (Stokes step + SuperLU nnz) on the box host, written straight into gpurun_out/golden;
# meanwhile the GPU runs the bench (no CPU baseline: the host is busy), the gyroid workload and increment counts.
mkdir -p gpurun_out/golden
( PMNS_GOLDEN_DIR=gpurun_out/golden timeout 3000 python scripts/oracle_golden.py cfg3 stokes nnz > gpurun_out/golden/cfg3_golden.log 2>&1 ) &
OPID=$!
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3_c.json 2> gpurun_out/bench_cfg3_c.err
PMNS_VERBOSE=1 timeout 400 python scripts/run_config.py gyroid 2>&1 | grep -v "fgmres\|pmns nd\|gputime\|newton\]" > gpurun_out/gyroid_gpu.log
bash scripts/exp_r2f.sh
wait $OPID
