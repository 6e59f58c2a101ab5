#!/bin/bash
mkdir -p gpurun_out
PMNS_VERBOSE=1 timeout 1500 python scripts/run_transient_check.py cfg4h > gpurun_out/r_cfg4h.txt 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r_bench_reference.json 2> gpurun_out/r_bench_reference.err; echo "rc=$?" >> gpurun_out/r_bench_reference.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/r_smoke.txt
