"""Per-rank frame time of the multi-GPU tile partition, measured on ONE GPU (developer tool).

The multi-GPU frame (parallel.py) gives tile k to rank k mod N and every rank
renders its share independently; only the final gather is a collective.  This tool renders the
share of every rank r of N, one after the other on the one GPU a gpurun call has, and reports
max_r t(r, N): the compute part of the N-GPU frame time.  The NCCL gather (16 B/pixel to rank 0)
is NOT in these numbers; a bound for it is printed beside them.

usage: python tools/sim_scaling.py [c3|c4s] [1080p|4k] ...
"""
import hashlib, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_1801_01155_b200 as lv
from paper_1801_01155_b200 import synth, parallel
from paper_1801_01155_b200.raycast import FramePlan

RES = {"1080p": (1920, 1080), "4k": (3840, 2160)}


def scene(name):
    dims = (256,) * 3
    n = {"c3": 100000, "c4s": 1000000}[name]
    lines = synth.turbulence(n, 100, dims)
    m = lv.build_voxel_model(lv.CurveSet.from_flat(*lines), lv.GridSpec(dims))
    oc = lv.build_lod(m)
    m.ao = lv.precompute_voxel_ao(m, oc)
    return dims, m, oc


def time_share(plan, W, H, reps):
    n_tiles = plan.n_my_tiles()
    img = torch.empty((max(n_tiles, 1), parallel.MG_TILE_H, parallel.MG_TILE_W, 4), dtype=torch.float32, device="cuda")
    st = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
    for _ in range(2):
        st.zero_()
        plan.launch(img, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.launch(img, st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, img


def main():
    args = sys.argv[1:]
    names = [a for a in args if a in ("c3", "c4s")] or ["c3"]
    ress = [a for a in args if a in RES] or ["1080p", "4k"]
    out = []
    for name in names:
        dims, m, oc = scene(name)
        for res in ress:
            W, H = RES[res]
            for label, kw in (("alpha .25 + precomputed AO", dict(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed")),
                              ("alpha .25 + precomputed AO + cone shadows",
                               dict(base_opacity=0.25, neighbor_mode="on", ao_mode="precomputed", shadow_mode="cone",
                                    light_dir=(0.3, 0.2, 1.0))))[:1 if os.environ.get("SIM_QUICK") else 2]:
                cam = lv.default_camera(dims, W, H)
                p = lv.RenderParams(**kw)
                base = None
                for N in [int(x) for x in os.environ.get('SIM_N', '1,2,4,8').split(',')]:
                    ts = []
                    for r in range(N):
                        plan = FramePlan(cam, m, oc, p, 1, tile_first=r, tile_step=N, compact=True,
                                         tile_w=parallel.MG_TILE_W, tile_h=parallel.MG_TILE_H)
                        t, _ = time_share(plan, W, H, 3)
                        ts.append(t)
                    worst = max(ts)
                    base = base or worst
                    gather_ms = 16.0 * W * H * (N - 1) / N / 900e9 * 1e3  # inbound to rank 0 at 900 GB/s
                    row = dict(scene=name, res=res, mode=label, n_ranks=N, max_rank_ms=round(worst, 3),
                               min_rank_ms=round(min(ts), 3), speedup_compute=round(base / worst, 2),
                               gather_bound_ms=round(gather_ms, 3),
                               speedup_with_gather_bound=round(base / (worst + gather_ms), 2))
                    out.append(row)
                    print(json.dumps(row), flush=True)
    return out


if __name__ == "__main__":
    main()
