#!/bin/bash
# quick A/B of the frame engines: correctness on tiny+small (wavefront == tile), then C3 timings + hashes
out=gpurun_out; mkdir -p $out
timeout 300 python tools/wf_check.py tiny 2>&1 | tail -8
timeout 300 python tools/wf_check.py small 2>&1 | tail -3
PERF_QUICK=1 timeout 600 python tools/frame_perf.py ${1:-c3} 2>&1 | tail -4
