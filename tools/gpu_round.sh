#!/bin/bash
# One GPU-box visit: parity tests, bench line, ncu launch list and one full capture of the frame kernel.
# usage: gpurun --timeout 1500 -- 'bash tools/gpu_round.sh <tag>'
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/smi_$tag.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" | tee -a $out/pytest_gpu_$tag.log
tail -3 $out/pytest_gpu_$tag.log
timeout 600 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?"
cat $out/bench_$tag.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err; echo "bench ref rc=$?"
cat $out/bench_ref_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
# one whole wavefront frame (every wf_* kernel of the first frame after the stages) ...
PERF_QUICK=1 timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy --section InstructionStats --clock-control none -k regex:wf_ -c 130 -f -o $out/prof_wf_$tag \
    python tools/frame_perf.py c3 > $out/ncu_wf_$tag.log 2>&1; echo "ncu wavefront rc=$?"
# ... and the tile kernel (own-voxel frames and the footprint pass use it)
LVX_ENGINE=tile timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -f -o $out/prof_render_$tag \
    python bench.py --steps 2 --warmup 3 --no-cpu > $out/ncu_full_$tag.log 2>&1; echo "ncu full rc=$?"
