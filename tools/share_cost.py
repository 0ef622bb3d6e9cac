import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200.raycast import FramePlan
from sim_scaling import scene, time_share
dims, m, oc = scene("c3")
W, H = 1920, 1080
cam = lv.default_camera(dims, W, H)
p = lv.RenderParams(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
plan = FramePlan(cam, m, oc, p, 1, tile_first=N // 2, tile_step=N, compact=True, tile_w=32, tile_h=16)
t, _ = time_share(plan, W, H, 3)
print("N", N, "tiles", plan.n_my_tiles(), "ms %.3f" % t, flush=True)
