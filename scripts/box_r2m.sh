#!/bin/bash
# Sub-phase trace of a warm config-3 build (M_d after M_p so the spans are clean), then the transient pipeline on
# half of config 4 with the oracle's residual check.
mkdir -p gpurun_out
PMNS_MD_AFTER=1 timeout 600 python scripts/trace_build.py cfg3 2 > gpurun_out/m_trace_build_cfg3.txt 2>&1
timeout 2400 python scripts/run_transient_check.py cfg4h > gpurun_out/m_cfg4h.txt 2>&1
