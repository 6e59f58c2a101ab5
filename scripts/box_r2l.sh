#!/bin/bash
# Per-kernel device time of one warm config-3 build (ncu launch list) + the Gyroid at h_m = 0.75 (serial build)
mkdir -p gpurun_out
timeout 600 python scripts/profile_build.py cfg3 > gpurun_out/l_profile_build_plain.txt 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/l_build_launches.csv python scripts/profile_build.py cfg3 > gpurun_out/l_profile_build_ncu.txt 2>&1
gzip -f gpurun_out/l_build_launches.csv
