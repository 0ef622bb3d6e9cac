#!/bin/bash
# Time every build/variants/*.so on a scene (developer tool; run under gpurun).
scene=${1:-c3}
export PERF_QUICK=1
for so in build/variants/*.so; do
  echo "== $so"
  LVX_LIB=$PWD/$so timeout 300 python tools/frame_perf.py $scene 2>&1 | tail -2
done
