#!/bin/bash
# nested-dissection leaf size vs stored M_p bytes, apply time and build time (Stokes step)
R=scripts/run_config.py
L=gpurun_out/exp_leaf.log
for leaf in 256 128 64; do
  for c in "cfg2" "cfg3 ws_merge_h=1.0"; do
    echo "== leaf=$leaf $c" >> $L
    PMNS_ND_LEAF=$leaf PMNS_MD_LEAF=$leaf timeout 300 python $R $c max_newton=1 >> $L 2>&1
  done
done
