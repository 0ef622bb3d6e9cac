#!/bin/bash
# correctness (wavefront == tile on the small scenes) of the in-tree library, then A/B of build/variants/{base,$1}.so (developer tool)
bash tools/r2_quick.sh c3 2>&1 | grep -E "^OK|FAIL|differ|Error|error|Traceback" | head
for rep in 1 2; do
for so in base ${1:-new}; do
  echo "== $so"
  LVX_LIB=$PWD/build/variants/$so.so PERF_QUICK=1 timeout 300 python tools/frame_perf.py c3 2>&1 | grep -E "nb a|own a" | sed 's/S=9683143//; s/stats.*//'
  LVX_LIB=$PWD/build/variants/$so.so timeout 300 python tools/share_frames.py 8 1080p | tail -1
  LVX_LIB=$PWD/build/variants/$so.so timeout 300 python tools/share_frames.py 8 4k | tail -1
done
done
