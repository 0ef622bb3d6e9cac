"""Small frames through the wavefront engine: time and final queue scale (developer tool)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from paper_1801_01155_b200.raycast import FramePlan
dims = (64,) * 3
m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.helices(1000, 100, dims)), lv.GridSpec(dims))
oc = lv.build_lod(m)
for (W, H) in ((64, 64), (256, 256), (640, 360)):
    for kw in (dict(neighbor_mode="on"), dict(base_opacity=0.1, neighbor_mode="on"), dict(base_opacity=0.02, tau=1.0, neighbor_mode="on")):
        cam = lv.default_camera(dims, W, H)
        plan = FramePlan(cam, m, oc, lv.RenderParams(**kw), 1, engine="wavefront")
        img = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
        st = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
        plan.launch(img, st)
        s0 = plan._scale
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.launch(img, st)
        e1.record()
        torch.cuda.synchronize()
        print(f"{W}x{H} {kw}: scale after first launch {s0}, {e0.elapsed_time(e1) / 10:.3f} ms", flush=True)
