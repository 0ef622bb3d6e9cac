#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q -k "ao or lod or smoke or density" 2>&1 | tail -3
timeout 600 python tools/ao_perf.py 2>&1 | tail -6
LVX_AO_LEGACY=1 timeout 600 python tools/ao_perf.py 2>&1 | tail -3
