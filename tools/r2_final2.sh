#!/bin/bash
# final evidence of round 2, second session: GPU tests, bench line (both arms), full ncu tables of one
# frame (second frame of tools/frame_perf.py: 2 + 10 x 5 launches once the first burst is sized by the
# previous frame) and of the preprocessing stages, launch list of the default bench command
tag=${1:-r2n}; out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; tail -2 $out/pytest_gpu_$tag.log
timeout 800 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref_$tag.json 2> $out/bench_ref_$tag.err; echo "bench ref rc=$?"
WF_SKIP=62 WF_COUNT=52 SKIP_SRC=1 bash tools/r2_ncu_all.sh $tag
python tools/ncu_table.py $out/wf_raw_$tag.csv --title "one C3 1080p wavefront frame (52 launches), final round-2 kernels ($tag)" --out $out/${tag}_wavefront_kernels.txt --json $out/${tag}_traffic.json
python tools/ncu_table.py $out/stages_raw_$tag.csv --title "preprocessing stages of C3, final round-2 kernels ($tag; two passes)" --out $out/${tag}_stage_kernels.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-targets --no-variants > $out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
rm -f $out/wf_raw_$tag.csv $out/stages_raw_$tag.csv
cut -c1-150 $out/${tag}_wavefront_kernels.txt; cut -c1-150 $out/${tag}_stage_kernels.txt
