#!/bin/bash
mkdir -p gpurun_out
timeout 600 python scripts/memplan.py cfg3 1.0:25 > gpurun_out/u_memplan_cfg3.txt 2>&1
timeout 600 python scripts/memplan.py cfg4 0.5:50 > gpurun_out/u_memplan_cfg4.txt 2>&1
timeout 300 python scripts/memplan.py cfg2 0.5:50 > gpurun_out/u_memplan_cfg2.txt 2>&1
