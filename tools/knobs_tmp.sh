export LVX_LIB=$PWD/build/variants/k4.so SIM_QUICK=1 SIM_N=1,8
run() { echo "== $*"; env "$@" python tools/sim_scaling.py c3 1080p 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(r['n_ranks'], r['max_rank_ms'])"; }
run X=1
run LVX_WF_TAIL_RAYS=4000 LVX_WF_TAIL_BITS=2
run LVX_WF_TAIL_RAYS=4000 LVX_WF_TAIL_BITS=4
run LVX_WF_TAIL_RAYS=30000 LVX_WF_TAIL_BITS=2
run LVX_WF_TAIL_RAYS=30000 LVX_WF_TAIL_BITS=4
run LVX_WF_GROW=7 LVX_WF_GROW_BITS=1
run LVX_WF_GROW=5 LVX_WF_GROW_BITS=1
