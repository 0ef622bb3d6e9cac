#!/bin/bash
# ray-kernel grid size against the slowest 1-of-N share (developer tool)
run() { echo "== $*"; env "$@" SIM_N=${SIMN:-1,2,8} SIM_QUICK=1 timeout 600 python tools/sim_scaling.py c3 4k 1080p 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('  ', d['res'], d['n_ranks'], d['max_rank_ms'], d['speedup_compute'])"; }
for g in 2 3 4 6 8; do run LVX_WF_GRID_RAYS=$g; done
