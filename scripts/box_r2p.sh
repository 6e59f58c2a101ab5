#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scripts/trace_solve.py cfg3 > gpurun_out/p_trace_solve_cfg3.txt 2>&1
