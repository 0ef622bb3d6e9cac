#!/bin/bash
# Stage the reference's own hot-path test files where a GPU box can see them: baseline/_ref/ is
# git-ignored (nothing of the reference enters the history) but travels with gpurun.
set -e
cd "$(dirname "$0")/.."
mkdir -p baseline/_ref/tests
for f in test_voxelizer.py test_lod.py test_raycast.py test_illumination.py; do
    cp /root/reference/pkg/tests/$f baseline/_ref/tests/$f
done
ls -la baseline/_ref/tests
