#!/bin/bash
# per-kernel time split of one C3 wavefront frame, caches NOT flushed between kernels (developer tool)
out=gpurun_out; mkdir -p $out
PERF_QUICK=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:wf_ -c ${WF_N:-200} --csv --log-file $out/wf_launches_raw_${1:-x}.csv python tools/frame_perf.py c3 > $out/ncu_raw_${1:-x}.log 2>&1; echo "ncu rc=$?"
