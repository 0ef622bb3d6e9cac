"""One wavefront frame of a bench scene with LVX_WF_DEBUG counters (developer tool)."""
import os, sys
os.environ["LVX_WF_DEBUG"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from paper_1801_01155_b200.raycast import FramePlan
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
nbm = sys.argv[2] if len(sys.argv) > 2 else "on"
dims = (256,) * 3
lines = synth.turbulence(100000 if name == "c3" else 1000000, 100, dims)
m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(dims))
oc = lv.build_lod(m)
m.ao = lv.precompute_voxel_ao(m, oc)
cam = lv.default_camera(dims, 1920, 1080)
p = lv.RenderParams(base_opacity=0.25, neighbor_mode=nbm, ao_mode="precomputed")
plan = FramePlan(cam, m, oc, p, 1 if nbm == "on" else 0, engine="wavefront")
img = torch.empty((1080, 1920, 4), dtype=torch.float32, device="cuda")
st = torch.zeros((1080, 3), dtype=torch.int64, device="cuda")
plan.launch(img, st)
torch.cuda.synchronize()
