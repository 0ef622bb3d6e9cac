"""Where render_frame's host-side time goes (developer tool)."""
import cProfile, pstats, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch
import paper_1801_01155_b200 as lv
from frame_perf import scene
dims, m, oc = scene("c3")
cam = lv.default_camera(dims, 1920, 1080)
p = lv.RenderParams(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed")
for _ in range(3):
    fr = lv.render_frame(cam, m, oc, None, p)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    fr = lv.render_frame(cam, m, oc, None, p)
torch.cuda.synchronize()
print("render_frame %.3f ms/frame, kernel %.3f ms" % ((time.perf_counter() - t0) * 50, fr.stats["ms"]))
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    fr = lv.render_frame(cam, m, oc, None, p)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(40)
