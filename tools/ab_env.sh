#!/bin/bash
# correctness of the in-tree library on the small scenes, then A/B of one environment switch on the full C3 frame and
# on 1-of-8 shares (developer tool): tools/ab_env.sh VAR a b
bash tools/r2_quick.sh c3 2>&1 | grep -E "^OK|FAIL|differ|Error|error|Traceback" | head
for rep in 1 2; do
for v in $2 $3; do
  echo "== $1=$v"
  env $1=$v PERF_QUICK=1 timeout 300 python tools/frame_perf.py c3 2>&1 | grep -E "nb a|own a" | sed 's/S=9683143//; s/stats.*//'
  env $1=$v timeout 300 python tools/share_frames.py 8 1080p | tail -1
  env $1=$v timeout 300 python tools/share_frames.py 8 4k | tail -1
done
done
