#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "packed or encoded" 2>&1 | tail -4
for r in rec packed; do echo "== LVX_RECORDS=$r"; PERF_QUICK=1 LVX_RECORDS=$r timeout 300 python tools/frame_perf.py c3 2>&1 | grep "nb a"; done
for r in rec packed; do echo "== c4s LVX_RECORDS=$r"; PERF_QUICK=1 LVX_RECORDS=$r timeout 600 python tools/frame_perf.py c4s 2>&1 | grep "nb a"; done
