#!/bin/bash
mkdir -p gpurun_out
for mb in 5 6 8; do
  PMNS_JAC_MINB=$mb timeout 600 python scripts/bench_jacobian.py cfg4 30 > gpurun_out/x_jbench_minb$mb.json 2> gpurun_out/x_jbench_minb$mb.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -q -x -k "operators or assembly or jacobian or jrec or residual" > gpurun_out/x_optest.log 2>&1; echo "rc=$?" >> gpurun_out/x_optest.log
