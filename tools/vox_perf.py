"""Voxelizer timing on a bench line set (developer tool): stage-by-stage CUDA-event times."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth, _lib

def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    if name == "c3":
        dims = (256,) * 3; lines = synth.turbulence(100000, 100, dims)
    elif name == "c2":
        dims = (128,) * 3; lines = synth.helices(10000, 100, dims)
    elif name == "c4s":
        dims = (256,) * 3; lines = synth.turbulence(1000000, 100, dims)
    pts, attrs, off = lines
    spec = lv.GridSpec(dims, 32)
    pts_d, attrs_d, off_d = _lib.to_device(pts), _lib.to_device(attrs), _lib.to_device(off)
    n = int(off.size - 1)
    out = lv.voxelize_device(pts_d, attrs_d, off_d, n, spec, caches=False, provenance=False)
    S = out["n_segments"]
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        out = lv.voxelize_device(pts_d, attrs_d, off_d, n, spec, caches=False, provenance=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    import hashlib
    h = hashlib.sha256(out["packed"].cpu().numpy().tobytes()).hexdigest()[:16]
    P = pts.shape[0]
    b = 32 * P + S * 31 + 5 * spec.voxel_count
    t = min(ts)
    print(f"[{name}] S={S} dropped={out['dropped']} voxelize min {t:.3f} ms  median {sorted(ts)[len(ts)//2]:.3f} ms "
          f"{S/t/1e3:.0f} Mseg/s  {b/t/1e6:.0f} GB/s  packed {h}", flush=True)

main()
