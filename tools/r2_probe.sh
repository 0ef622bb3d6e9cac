#!/bin/bash
# round-2 first probe: tests, per-iteration counters, raw per-launch list of two frames
out=gpurun_out; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_r2a.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_r2a.log
timeout 600 python tools/wf_iters.py c3 > $out/wf_iters_r2a.log 2>&1; echo "iters rc=$?"; tail -20 $out/wf_iters_r2a.log
PERF_QUICK=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:wf_ -c 200 --csv --log-file $out/wf_launches_raw_r2a.csv python tools/frame_perf.py c3 > $out/ncu_raw_r2a.log 2>&1; echo "ncu rc=$?"
PERF_QUICK=1 timeout 600 python tools/frame_perf.py c3 2>&1 | tail -5
