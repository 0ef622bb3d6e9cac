#!/bin/bash
# full-set ncu captures, exported to CSV on the box (the .ncu-rep files of a whole frame exceed what
# gpurun copies back): one wavefront frame (second frame of tools/frame_perf.py), the stage kernels, and
# small source-level captures of one iteration / one pass.
# usage: gpurun --timeout 3000 -- 'bash tools/r2_ncu_all.sh <tag>'
tag=${1:-r2a}; out=gpurun_out; mkdir -p $out; tmp=/tmp/ncu_$tag; mkdir -p $tmp
STAGE_RE='regex:clip_|regroup|compact|scan_|density_l0|mip_|mip3|ao_bake|count_crossings|nsum|emit_|vox_|mark_starts'
PERF_QUICK=1 timeout 1500 ncu --set full --clock-control none -k regex:wf_ -s ${WF_SKIP:-62} -c ${WF_COUNT:-62} -f -o $tmp/wf \
    python tools/frame_perf.py c3 > $out/ncu_wf_$tag.log 2>&1; echo "ncu wavefront rc=$?"
ncu -i $tmp/wf.ncu-rep --page raw --csv > $out/wf_raw_$tag.csv 2>/dev/null; rm -f $tmp/wf.ncu-rep
if [ -z "$SKIP_STAGES" ]; then
timeout 1500 ncu --set full --clock-control none -k "$STAGE_RE" -s ${ST_SKIP:-0} -c ${ST_COUNT:-80} -f -o $tmp/st \
    python tools/stage_run.py > $out/ncu_stages_$tag.log 2>&1; echo "ncu stages rc=$?"
ncu -i $tmp/st.ncu-rep --page raw --csv > $out/stages_raw_$tag.csv 2>/dev/null; rm -f $tmp/st.ncu-rep
fi
if [ -z "$SKIP_SRC" ]; then
# source-level: the wf kernels of iteration 1 of the second frame, and one launch of each heavy stage kernel
PERF_QUICK=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:wf_ -s ${WF_SRC_SKIP:-69} -c ${WF_SRC_COUNT:-4} -f -o $out/src_wf_$tag \
    python tools/frame_perf.py c3 > $out/ncu_wfsrc_$tag.log 2>&1; echo "ncu wf source rc=$?"
if [ -z "$SKIP_STAGES" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "${ST_SRC_RE:-regex:clip_|regroup_kernel|compact_kernel|density_l0|ao_bake|emit_}" -s ${ST_SRC_SKIP:-9} -c ${ST_SRC_COUNT:-5} -f -o $out/src_stages_$tag \
    python tools/stage_run.py > $out/ncu_stsrc_$tag.log 2>&1; echo "ncu stage source rc=$?"
fi
fi
ls -la $out | tail -20; du -sh $out
