#!/bin/bash
# ncu full capture of the frame kernel on one bench scene (developer tool).
# usage: gpurun -- 'bash tools/prof_frame.sh <tag> [scene] [case-index]'
tag=${1:-x}; scene=${2:-c3}; 
export PERF_QUICK=1
timeout 600 python tools/frame_perf.py $scene 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 2 -c 1 -f -o gpurun_out/prof_render_$tag \
    python tools/frame_perf.py $scene > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu rc=$?"
