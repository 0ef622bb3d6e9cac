"""Runs every preprocessing stage of the C3 scene twice (developer tool; what ncu profiles).
Launch order per pass: mark_starts, count_crossings, clip, scan x3, regroup, compact | density_l0 | mip x N | ao_bake"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth, _lib
from paper_1801_01155_b200.illumination import ao_bake_device
from paper_1801_01155_b200.lod import density_level0_device, mips_inplace, octree_buffer

dims = (256,) * 3
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
pts, attrs, off = synth.turbulence(n, 100, dims)
spec = lv.GridSpec(dims, 32)
pts_d, attrs_d, off_d = _lib.to_device(pts), _lib.to_device(attrs), _lib.to_device(off)
model = lv.build_voxel_model(lv.CurveSet.from_flat(pts, attrs, off), spec)
octree = lv.build_lod(model)
torch.cuda.synchronize()
print("== passes start", flush=True)
for rep in range(2):
    lv.voxelize_device(pts_d, attrs_d, off_d, n, spec, caches=False, provenance=False)
    flat, v0 = octree_buffer(dims)
    density_level0_device(model, out=flat[:v0])
    mips_inplace(flat, dims)
    ao_bake_device(model, octree, lv.AOParams(n_rays=100, radius=5.0, step=1.0))
    torch.cuda.synchronize()
print("done")
