#!/bin/bash
# final round-2 evidence: full ncu tables (frame, stages), source-level captures, the packed-record variant
tag=${1:-r2f}; out=gpurun_out
bash tools/r2_ncu_all.sh $tag
# the pre-reject / exact kernels reading the encoded records instead of the 32-byte render records (iteration 1)
tmp=/tmp/ncu_$tag
LVX_RECORDS=packed PERF_QUICK=1 timeout 900 ncu --set full --clock-control none -k regex:"wf_cand|wf_exact" -s 26 -c 2 -f -o $tmp/pk \
    python tools/frame_perf.py c3 > $out/ncu_pk_$tag.log 2>&1; echo "ncu packed rc=$?"
ncu -i $tmp/pk.ncu-rep --page raw --csv > $out/wf_packed_raw_$tag.csv 2>/dev/null; rm -f $tmp/pk.ncu-rep
LVX_RECORDS=rec PERF_QUICK=1 timeout 900 ncu --set full --clock-control none -k regex:"wf_cand|wf_exact" -s 26 -c 2 -f -o $tmp/rc \
    python tools/frame_perf.py c3 > $out/ncu_rc_$tag.log 2>&1; echo "ncu rec rc=$?"
ncu -i $tmp/rc.ncu-rep --page raw --csv > $out/wf_rec_raw_$tag.csv 2>/dev/null; rm -f $tmp/rc.ncu-rep
# launch list of the default bench command (shares of the step)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-targets --no-variants > $out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
du -sh $out
