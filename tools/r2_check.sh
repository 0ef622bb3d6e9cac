#!/bin/bash
# tests + default bench + reference arm (what the driver runs at round end)
tag=${1:-r2}; out=gpurun_out; mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -x -q > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"; tail -5 $out/pytest_gpu_$tag.log
timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?"; tail -3 $out/bench_$tag.err
cat $out/bench_$tag.json
