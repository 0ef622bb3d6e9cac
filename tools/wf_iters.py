"""Per-iteration counters of one wavefront frame (developer tool): LVX_WF_DEBUG=1 output."""
import os, sys
os.environ["LVX_WF_DEBUG"] = "1"  # (read once per process by the library)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200.raycast import FramePlan
sys.path.insert(0, os.path.join(ROOT, "tools"))
from sim_scaling import scene  # noqa
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
dims, m, oc = scene(name)
cam = lv.default_camera(dims, 1920, 1080)
p = lv.RenderParams(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed")
plan = FramePlan(cam, m, oc, p, 1)
img = torch.empty((1080, 1920, 4), dtype=torch.float32, device="cuda")
st = torch.zeros((1080, 3), dtype=torch.int64, device="cuda")
plan.launch(img, st)
torch.cuda.synchronize()
st.zero_()
plan.launch(img, st)
torch.cuda.synchronize()
