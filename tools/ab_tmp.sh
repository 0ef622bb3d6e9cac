export PERF_QUICK=1
for g in 8 12 16 24 32 64; do
  echo "-- grid mult $g"; LVX_WF_GRID_RAYS=$g python tools/frame_perf.py c3 2>&1 | grep "nb a.25"
  for n in 8; do LVX_WF_GRID_RAYS=$g python tools/fixed_cost_tmp.py $n; done
done
