export PMNS_VERBOSE=1
for extra in "body_force=0,0,0 p_in=3000" "body_force=2600,0,0 p_in=0 ws_merge_h=0.5" ; do
  echo "=== $extra"
  timeout 600 python scripts/run_config.py cfg3 ws_merge_h=0.25 ws_min_cells=50 max_newton=1 max_krylov=300 $extra 2>&1 | grep -E "fgmres\] it (25|50|100|200|300) |config" | cut -c1-300
done
