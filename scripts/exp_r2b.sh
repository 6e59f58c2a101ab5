#!/bin/bash
L=gpurun_out/exp_r2b.log
echo "== jacobian cfg4 (4 threads per record)" >> $L
timeout 300 python scripts/bench_jacobian.py cfg4 40 >> $L 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "jacobian_cell_records or operators" >> $L 2>&1
bash scripts/exp_leaf.sh
