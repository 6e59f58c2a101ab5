#!/bin/bash
# Round 2 (session 3) first box call: config-3 oracle goldens (Stokes step at h_m = 1.0 + SuperLU nnz) on the box
# host in the background (they need more host memory than the build container has); meanwhile the GPU runs the
# test suite and a config-3 bench line (CPU baseline skipped: the host is busy with the oracle).
mkdir -p gpurun_out/golden
( nproc; free -g; lscpu | grep "Model name" ) > gpurun_out/golden/host.txt 2>&1
( PMNS_GOLDEN_DIR=gpurun_out/golden timeout ${GOLDEN_S:-4500} python scripts/oracle_golden.py cfg3 stokes nnz \
    > gpurun_out/golden/cfg3_golden.log 2>&1; free -g >> gpurun_out/golden/cfg3_golden.log ) &
OPID=$!
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity.py::test_cfg3_stokes_step_full_size \
    > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
echo "bench rc=$?" >> gpurun_out/bench_cfg3.err
wait $OPID
