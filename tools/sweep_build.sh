#!/bin/bash
# Build variants of the library with different -D knobs (developer tool).
# usage: tools/sweep_build.sh name1 "-DA=1 -DB=2" name2 "..." ...   -> build/variants/<name>.so
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
S=paper_1801_01155_b200/csrc
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -ftz=false \
    -Xcompiler -fPIC -shared $flags $S/lvx_api.cu $S/lvx_voxelize.cu $S/lvx_lod.cu $S/lvx_render.cu $S/lvx_wavefront.cu $S/lvx_ao.cu $S/lvx_rep.cu $S/lvx_brute.cu -o build/variants/$name.so &
done
wait
ls -la build/variants
