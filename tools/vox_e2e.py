"""Where build_voxel_model's host-arrays-in / model-out time goes (developer tool)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth, _lib, voxelizer as vz

dims = (256,) * 3
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
pts, attrs, off = synth.turbulence(n, 100, dims)
spec = lv.GridSpec(dims, 32)


def T(label, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label:40s} {(time.perf_counter() - t0) * 1e3:9.2f} ms", flush=True)
    return r


for rep in range(3):
    print("--- rep", rep)
    cs = T("CurveSet.from_flat (validation)", lambda: lv.CurveSet.from_flat(pts, attrs, off))
    T("build_voxel_model total", lambda: lv.build_voxel_model(cs, spec))
    pts_d = T("H2D pts (pageable)", lambda: _lib.to_device(pts, np.float64))
    attrs_d = T("H2D attrs", lambda: _lib.to_device(attrs, np.float64))
    off_d = T("H2D off", lambda: _lib.to_device(off, np.int64))
    nc = int(off.size - 1)
    T("voxelize_device caches+provenance", lambda: vz.voxelize_device(pts_d, attrs_d, off_d, nc, spec))
    T("voxelize_device bare", lambda: vz.voxelize_device(pts_d, attrs_d, off_d, nc, spec, caches=False, provenance=False))
    out = vz.voxelize_device(pts_d, attrs_d, off_d, nc, spec)
    m = T("model_from_device", lambda: vz.model_from_device(out, spec, vz.default_transfer_table()))
    T("stage_clip", lambda: vz.stage_clip(pts_d, attrs_d, off_d, nc, spec, True))

# --- where the time inside build_voxel_model goes: wrap its steps ---------------------------
import time as _t
acc = {}
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = _t.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + (_t.perf_counter() - t0) * 1e3
        return r
    setattr(mod, name, g)
for n in ("stage_clip", "stage_scan", "stage_regroup", "stage_compact", "stage_provenance", "model_from_device", "voxelize_device"):
    wrap(vz, n)
wrap(_lib, "to_device")
cs = lv.CurveSet.from_flat(pts, attrs, off)
for rep in range(2):
    acc.clear()
    torch.cuda.synchronize(); t0 = _t.perf_counter()
    m = lv.build_voxel_model(cs, spec)
    torch.cuda.synchronize()
    print("build_voxel_model %.2f ms:" % ((_t.perf_counter() - t0) * 1e3), {k: round(v, 2) for k, v in acc.items()})
    del m
