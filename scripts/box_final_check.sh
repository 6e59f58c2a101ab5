#!/bin/bash
# Quick check of the committed tree on a B200: smoke() and the non-slow GPU tests.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.txt
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x --deselect tests/test_gpu_parity.py::test_cfg2_end_to_end > gpurun_out/final_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/final_gputest.log
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "rc=$?" >> gpurun_out/final_bench.err
