#!/bin/bash
# cand / exact kernels of iteration 1 of the second C3 frame, reading the 32-byte render records vs the encoded records
tag=${1:-r2f}; out=gpurun_out; tmp=/tmp/ncu_$tag; mkdir -p $tmp
for r in rec packed; do
LVX_RECORDS=$r PERF_QUICK=1 timeout 900 ncu --set full --clock-control none -k regex:"wf_cand|wf_exact" -s 39 -c 3 -f -o $tmp/$r \
    python tools/frame_perf.py c3 > $out/ncu_${r}_$tag.log 2>&1; echo "ncu $r rc=$?"
ncu -i $tmp/$r.ncu-rep --page raw --csv > $out/wf_${r}_raw_$tag.csv 2>/dev/null; rm -f $tmp/$r.ncu-rep
done
