"""Quick frame timing + image hash on the bench scenes (developer tool)."""
import hashlib, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from paper_1801_01155_b200.raycast import FramePlan

def scene(name):
    if name == "c3":
        dims = (256,)*3; lines = synth.turbulence(100000, 100, dims)
    elif name == "c2":
        dims = (128,)*3; lines = synth.helices(10000, 100, dims)
    elif name == "c4s":  # 1M-line set of config 4 (single GPU, 1080p)
        dims = (256,)*3; lines = synth.turbulence(1000000, 100, dims)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    m.ao = lv.precompute_voxel_ao(m, oc)
    return dims, m, oc

NAMES = {0: "W walk", 1: "V headers", 2: "C pre-reject", 3: "E exact", 4: "insert", 5: "S list+shade", 6: "S accumulate",
         7: "tail", 8: "loop top", 9: "S decide", 10: "#rounds", 11: "#C chunks", 12: "#E batches", 13: "#S iters",
         14: "sum items", 15: "sum candidates", 16: "sum survivors", 17: "#S stages", 18: "sum shaded", 19: "#blocks"}

def dump_stage_clocks(quiet=False):
    import ctypes
    from paper_1801_01155_b200 import _lib
    L = _lib.lib()
    if not hasattr(L, "lvx_debug_stage_clocks"):
        return
    buf = (ctypes.c_uint64 * 32)()
    L.lvx_debug_stage_clocks(buf)
    v = list(buf)
    if quiet:
        return
    tot = sum(v[:10]) or 1
    for k in range(10):
        print(f"   clk {NAMES[k]:14s} {v[k]/tot*100:5.1f}%  {v[k]/max(v[19],1):12.0f} cyc/block")
    for k in range(10, 20):
        print(f"   cnt {NAMES[k]:14s} {v[k]/5:14.0f} /frame  {v[k]/max(v[19],1):10.2f} /block")

def main():
    names = sys.argv[1:] or ["c3"]
    for name in names:
        dims, m, oc = scene(name)
        cases = (("nb a.25 AO", dict(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed")),
                          ("own a.25 AO", dict(base_opacity=0.25, neighbor_mode="off", ao_mode="precomputed")),
                          ("nb a.25 AO cone", dict(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed", shadow_mode="cone", light_dir=(0.3, 0.2, 1.0))),
                          ("nb opaque", dict(neighbor_mode="on")))
        if os.environ.get("PERF_QUICK"):
            cases = cases[:2]
        for label, kw in cases:
            cam = lv.default_camera(dims, 1920, 1080)
            p = lv.RenderParams(**kw)
            plan = FramePlan(cam, m, oc, p, 1 if kw["neighbor_mode"] == "on" else 0)
            img = torch.empty((1080, 1920, 4), dtype=torch.float32, device="cuda")
            st = torch.zeros((1080, 3), dtype=torch.int64, device="cuda")
            for _ in range(2):
                plan.launch(img, st)
            torch.cuda.synchronize()
            dump_stage_clocks(quiet=True)
            st.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                plan.launch(img, st)
            e1.record()
            torch.cuda.synchronize()
            h = hashlib.sha256(img.cpu().numpy().tobytes()).hexdigest()[:12]
            dump_stage_clocks()
            print(f"[{name} {label}] S={m.segment_count} {e0.elapsed_time(e1)/5:.3f} ms  img {h} stats {(st.sum(0)//5).tolist()}", flush=True)

if __name__ == "__main__":
    main()
