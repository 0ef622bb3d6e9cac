#!/bin/bash
export PERF_QUICK=1
run() { echo "== $*"; env "$@" timeout 300 python tools/frame_perf.py c3 2>&1 | grep "nb a"; }
V=$PWD/build/variants
run LVX_LIB=$V/base.so
run LVX_LIB=$V/base.so LVX_WF_BUDGET=256
run LVX_LIB=$V/base.so LVX_WF_BUDGET=320
run LVX_LIB=$V/hs32.so LVX_WF_BUDGET=256
run LVX_LIB=$V/hs32.so LVX_WF_BUDGET=384
run LVX_LIB=$V/base.so LVX_WF_BUDGET=160
run LVX_LIB=$V/base.so
