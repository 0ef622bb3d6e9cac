#!/bin/bash
# compute-sanitizer over both frame engines + voxelizer / LoD / AO bake on a small scene
out=gpurun_out
for tool in memcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python tools/wf_check.py tiny > $out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|OK$|FAIL$" $out/sanitize_$tool.log | tail -3
done
