"""Renders the share of rank 0 of N of a C3 frame a few times (developer tool; what ncu lists)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import parallel
from paper_1801_01155_b200.raycast import FramePlan
from frame_perf import scene
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
W, H = (3840, 2160) if (len(sys.argv) > 2 and sys.argv[2] == "4k") else (1920, 1080)
dims, m, oc = scene("c3")
cam = lv.default_camera(dims, W, H)
p = lv.RenderParams(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed")
plan = FramePlan(cam, m, oc, p, 1, tile_first=0, tile_step=N, compact=True, tile_w=parallel.MG_TILE_W, tile_h=parallel.MG_TILE_H)
img = torch.empty((max(plan.n_my_tiles(), 1), parallel.MG_TILE_H, parallel.MG_TILE_W, 4), dtype=torch.float32, device="cuda")
st = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
for _ in range(4):
    plan.launch(img, st)
torch.cuda.synchronize()
import time
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t0 = time.perf_counter(); e0.record(); plan.launch(img, st); e1.record(); torch.cuda.synchronize()
    ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
print("share 1/%d %dx%d: events min %.3f ms median %.3f ms; wall min %.3f ms" % (N, W, H, min(t[0] for t in ts), sorted(t[0] for t in ts)[5], min(t[1] for t in ts)))
