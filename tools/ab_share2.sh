#!/bin/bash
# A/B of build/variants/*.so: full C3 frame and 1-of-8 shares at 1080p / 4K (developer tool)
for rep in 1 2; do
for so in build/variants/*.so; do
  echo "== $so"
  LVX_LIB=$PWD/$so PERF_QUICK=1 timeout 300 python tools/frame_perf.py c3 2>&1 | grep -E "nb a|own a" | sed 's/S=9683143//; s/stats.*//'
  LVX_LIB=$PWD/$so timeout 300 python tools/share_frames.py 8 1080p | tail -1
  LVX_LIB=$PWD/$so timeout 300 python tools/share_frames.py 8 4k | tail -1
done
done
