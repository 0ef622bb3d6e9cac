"""Wavefront engine vs tile engine on small scenes (developer tool): byte equality of
image and counters."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from paper_1801_01155_b200.raycast import FramePlan

def run(plan, W, H):
    img = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    st = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
    plan.launch(img, st)
    torch.cuda.synchronize()
    return img.cpu().numpy(), st.cpu().numpy()

def main():
    size = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    if size == "tiny":
        dims, n, P, W, H = (32,) * 3, 2000, 60, 320, 180
    elif size == "small":
        dims, n, P, W, H = (64,) * 3, 8000, 80, 640, 360
    else:
        dims, n, P, W, H = (128,) * 3, 10000, 100, 1920, 1080
    gen = synth.helices if size == "mid" else synth.turbulence
    lines = gen(n, P, dims)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    m.ao = lv.precompute_voxel_ao(m, oc, lv.AOParams(n_rays=16, radius=4.0, step=1.0))
    cases = [dict(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed"),
             dict(base_opacity=0.25, neighbor_mode="off", ao_mode="precomputed"),
             dict(neighbor_mode="on"),
             dict(base_opacity=0.05, tau=1.0, neighbor_mode="on"),
             dict(base_opacity=0.3, neighbor_mode="on", shadow_mode="cone", light_dir=(0.3, 0.2, 1.0)),
             dict(base_opacity=0.3, neighbor_mode="on", opacity_mode="distance-scaled", joint_spheres=False)]
    bad = 0
    for kw in cases:
        cam = lv.default_camera(dims, W, H)
        try:
            p = lv.RenderParams(**kw)
        except Exception as e:
            print("skip", kw, e); continue
        nb = 1 if kw["neighbor_mode"] == "on" else 0
        a = run(FramePlan(cam, m, oc, p, nb, engine="tile"), W, H)
        b = run(FramePlan(cam, m, oc, p, nb, engine="wavefront"), W, H)
        same_img = np.array_equal(a[0], b[0])
        same_st = np.array_equal(a[1], b[1])
        d = np.abs(a[0].astype(np.float64) - b[0]).max()
        print(f"{kw}: image {'==' if same_img else '!='} (max diff {d:.3e}, {int((a[0]!=b[0]).any(-1).sum())} px) "
              f"stats {'==' if same_st else '!='} tile {a[1].sum(0).tolist()} wf {b[1].sum(0).tolist()}", flush=True)
        bad += (not same_img) + (not same_st)
    print("FAIL" if bad else "OK")

main()
