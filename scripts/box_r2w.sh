#!/bin/bash
mkdir -p gpurun_out
for mb in 1 5 6; do
  PMNS_JAC_MINB=$mb timeout 600 python scripts/bench_jacobian.py cfg4 30 > gpurun_out/w_jbench_minb$mb.json 2> gpurun_out/w_jbench_minb$mb.err
done
