#!/bin/bash
# per-kernel time split of a 1-of-N share of the C3 frame (developer tool): wf_split_share.sh <N> <1080p|4k> <tag>
out=gpurun_out; mkdir -p $out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:wf_ -c 400 --csv --log-file $out/wf_share_raw_${3:-x}.csv python tools/share_frames.py ${1:-8} ${2:-4k} > $out/ncu_share_${3:-x}.log 2>&1; echo "ncu rc=$?"
python tools/wf_split.py $out/wf_share_raw_${3:-x}.csv 2
LVX_WF_DEBUG=1 python tools/share_frames.py ${1:-8} ${2:-4k} 2>&1 | grep "wf it" | tail -12 | cut -c1-200
