#!/bin/bash
# like ab_two.sh, with the cone-shadow and opaque frames as well (developer tool)
bash tools/r2_quick.sh c3 2>&1 | grep -E "^OK|FAIL|differ|Error|error|Traceback" | head
for rep in 1 2; do
for so in base ${1:-new}; do
  echo "== $so"
  LVX_LIB=$PWD/build/variants/$so.so timeout 300 python tools/frame_perf.py c3 2>&1 | grep -E "^\[c3" | sed 's/S=9683143//; s/stats.*//'
done
done
