"""LoD timing on the C3 / 1M-line scenes (developer tool)."""
import os, sys, hashlib
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth
from paper_1801_01155_b200.lod import density_level0_device, mips_inplace, octree_buffer
dims = (256,) * 3
for n in [int(x) for x in (sys.argv[1:] or ["100000"])]:
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*synth.turbulence(n, 100, dims)), lv.GridSpec(dims))
    flat, v0 = octree_buffer(dims)
    def ev(fn):
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        return min(ts)
    density_level0_device(m, out=flat[:v0])
    t0 = ev(lambda: density_level0_device(m, out=flat[:v0]))
    t1 = ev(lambda: mips_inplace(flat, dims))
    S, V = m.segment_count, m.voxel_count
    b = 25 * S + 4 * V + 4 * V * 9 / 7
    print(f"n={n} S={S}: density {t0:.4f} ms  mips {t1:.4f} ms  total {t0+t1:.4f} ms  {b/(t0+t1)/1e6:.0f} GB/s alg  hash {hashlib.sha256(flat.cpu().numpy().tobytes()).hexdigest()[:12]}", flush=True)
