#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --deselect tests/test_gpu_parity.py::test_cfg2_end_to_end > gpurun_out/y_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/y_gputest.log
for mb in 6 1; do
  PMNS_JAC_MINB=$mb timeout 600 python scripts/bench_jacobian.py cfg4 30 > gpurun_out/y_jbench_minb$mb.json 2> gpurun_out/y_jbench_minb$mb.err
done
