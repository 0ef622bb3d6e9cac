#!/bin/bash
# A/B of build/variants/*.so on the full C3 frame and on 1-of-8 shares (developer tool)
for so in build/variants/*.so; do
  echo "== $so"
  LVX_LIB=$PWD/$so PERF_QUICK=1 timeout 300 python tools/frame_perf.py c3 2>&1 | grep -E "nb a|own a" | sed 's/S=9683143//; s/stats.*//'
  LVX_LIB=$PWD/$so SIM_N=8 SIM_QUICK=1 timeout 600 python tools/sim_scaling.py c3 1080p 4k 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('   share', d['res'], d['n_ranks'], d['max_rank_ms'])"
done
