#!/bin/bash
# Allocator oversize-block reuse: traced warm config-3 build; config-4h transient with verbose build messages.
mkdir -p gpurun_out
PMNS_MD_AFTER=1 timeout 600 python scripts/trace_build.py cfg3 2 > gpurun_out/n_trace_build_cfg3.txt 2>&1
timeout 600 python scripts/trace_build.py cfg3 2 > gpurun_out/n_trace_build_cfg3_conc.txt 2>&1
PMNS_VERBOSE=1 PMNS_TRACE=1 timeout 2400 python scripts/run_transient_check.py cfg4h > gpurun_out/n_cfg4h.txt 2>&1
