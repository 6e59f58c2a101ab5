#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/bench_jacobian.py cfg4 30 > gpurun_out/z_jbench_ldcs.json 2> gpurun_out/z_jbench_ldcs.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -q -x -k "operators or assembly or jacobian or jrec or residual" > gpurun_out/z_optest.log 2>&1; echo "rc=$?" >> gpurun_out/z_optest.log
