#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --config cfg4h --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ae_bench_cfg4h.json 2> gpurun_out/ae_bench_cfg4h.err; echo "rc=$?" >> gpurun_out/ae_bench_cfg4h.err
