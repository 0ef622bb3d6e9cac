tag=${1:-r1e}; out=gpurun_out; mkdir -p $out
timeout 600 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
PERF_QUICK=1 timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats --section LaunchStats --section Occupancy --section InstructionStats --clock-control none -k regex:wf_ -c 130 -f -o $out/prof_wf_$tag \
    python tools/frame_perf.py c3 > $out/ncu_wf_$tag.log 2>&1; echo "ncu wavefront rc=$?"
LVX_ENGINE=tile timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -f -o $out/prof_render_$tag \
    python bench.py --steps 2 --warmup 3 --no-cpu > $out/ncu_full_$tag.log 2>&1; echo "ncu full rc=$?"
ls -la $out
