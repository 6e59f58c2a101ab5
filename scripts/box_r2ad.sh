#!/bin/bash
mkdir -p gpurun_out
( free -g | head -2 ) > gpurun_out/ad_memplan_cfg5.txt
PMNS_TRACE=1 timeout 2400 python scripts/memplan.py cfg5 0.5:50 >> gpurun_out/ad_memplan_cfg5.txt 2>&1
