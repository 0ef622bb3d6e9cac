"""AO bake timing on the C3 scene (developer tool)."""
import os, sys, hashlib
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from paper_1801_01155_b200.illumination import ao_bake_device
dims = (256,) * 3
m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(100000, 100, dims)), lv.GridSpec(dims))
oc = lv.build_lod(m)
for n_rays, radius in ((100, 5.0), (25, 3.0), (100, 8.0)):
    aop = lv.AOParams(n_rays=n_rays, radius=radius, step=1.0)
    ao_bake_device(m, oc, aop)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); out = ao_bake_device(m, oc, aop); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    f = out.flat_device() if hasattr(out, "flat_device") else out
    h = hashlib.sha256(f.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"AO bake n_rays={n_rays} R={radius}: {min(ts):.2f} ms  hash {h}", flush=True)
