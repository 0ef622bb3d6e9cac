#!/bin/bash
# env-knob sweep of the wavefront schedule on one scene (developer tool; run under gpurun)
export PERF_QUICK=1
run() { echo "== $*"; env "$@" timeout 300 python tools/frame_perf.py c3 2>&1 | grep "nb a"; }
V=$PWD/build/variants
run LVX_LIB=$V/base.so
run LVX_LIB=$V/wf24.so LVX_WF_WN=12
run LVX_LIB=$V/wf48.so LVX_WF_WN=12
run LVX_LIB=$V/wf48.so LVX_WF_WN=12 LVX_WF_WN_SHIFT=5
run LVX_LIB=$V/wf24.so LVX_WF_WN=12 LVX_WF_TAIL_FROM=4
run LVX_LIB=$V/wf24.so LVX_WF_WN=12 LVX_WF_TAIL_MODE=3
run LVX_LIB=$V/base.so LVX_WF_TAIL_FROM=4
run LVX_LIB=$V/base.so LVX_WF_TAIL_MODE=3
run LVX_LIB=$V/base.so LVX_WF_TAIL_MODE=2
