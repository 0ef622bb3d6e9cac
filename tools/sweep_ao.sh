#!/bin/bash
for so in build/variants/*.so; do echo "== $so"; LVX_LIB=$PWD/$so timeout 300 python tools/ao_perf.py 2>&1 | head -1; done
