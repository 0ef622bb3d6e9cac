"""render_frame end to end with the image in HBM + copy vs written straight to pinned host memory."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np, torch
import paper_1801_01155_b200 as lv
from sim_scaling import scene
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
dims, m, oc = scene(name)
for (W, H) in ((1920, 1080), (3840, 2160)):
    cam = lv.default_camera(dims, W, H)
    for kw in (dict(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed"), dict(base_opacity=0.25, neighbor_mode="off", ao_mode="precomputed")):
        p = lv.RenderParams(**kw)
        imgs = {}
        for mode in ("device", "host", "device", "host"):
            os.environ["LVX_FRAME_OUT"] = mode
            for _ in range(2):
                f = lv.render_frame(cam, m, oc, params=p)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ks = []
            for _ in range(10):
                f = lv.render_frame(cam, m, oc, params=p)
                ks.append(f.stats["ms"])
            dt = (time.perf_counter() - t0) / 10 * 1e3
            imgs[mode] = f.image.copy()
            print(f"{W}x{H} nb={kw['neighbor_mode']} out={mode}: e2e {dt:.3f} ms  kernel {np.mean(ks):.3f} ms", flush=True)
        print("   identical:", np.array_equal(imgs["device"], imgs["host"]))
