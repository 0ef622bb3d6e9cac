for so in build/variants/*.so; do echo "== $so"; LVX_LIB=$PWD/$so python tools/vox_perf.py c3 5 2>&1 | tail -1; done
