#!/bin/bash
for so in build/variants/*.so; do echo "== $so"; LVX_LIB=$PWD/$so timeout 300 python tools/lod_perf.py 100000 2>&1 | tail -1; done
