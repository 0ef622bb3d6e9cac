#!/usr/bin/env python
"""bench.py -- ms/frame of the linevox hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the config the metric "transparent+AO, 1080p"
is quoted on): 100k turbulence-like synthetic lines x 100 points, 256^3 grid,
N=32 bins -> 9.68 M segments; 1920x1080, alpha = 0.25, tau = 0.95, neighbour mode
on, precomputed LoD ambient occlusion (100 rays, radius 5).  A "step" is one frame.

* `value`    device time per frame (CUDA events around K frames, inputs resident in HBM).
* `e2e`      the same frame through the public API `render_frame` (`render_frame_tiled`
             for N > 1): camera/params from host objects, image copied back to pinned
             host memory and the counters read every step.
* `roofline` the frame kernel against the measured HBM peak, from the unique bytes the
             reference's algorithm touches (instrumented pass).
* `stages`   voxelize / LoD / AO bake timings of the same data set (Mseg/s, GB/s).
* `cpu_baseline` the CPU oracle (a C port of the reference, OpenMP) on every 8th-or-so
             row of the same frame.
N > 1: launched by torchrun; the image is split into interleaved tiles (strong scaling).
`--impl reference` times the CPU path only (the Python/numba reference cannot travel to
the GPU box; the pinned C port stands in).
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    # name: (generator, n_lines, pts, dims, W, H, RenderParams kwargs, AO bake)
    "c3": dict(gen="turbulence", n=100000, pts=100, dims=(256, 256, 256), W=1920, H=1080,
               params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed"),
               ao=(100, 5.0, 1.0),
               label="100k turbulence lines x100 pts, 256^3, 1080p transparent(alpha .25)+precomputed AO, neighbour on"),
    "c2": dict(gen="helices", n=10000, pts=100, dims=(128, 128, 128), W=1920, H=1080,
               params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on"), ao=None,
               label="10k helices x100 pts, 128^3, 1080p transparent(alpha .25), neighbour on"),
    "c1": dict(gen="helices", n=1000, pts=100, dims=(64, 64, 64), W=256, H=256,
               params=dict(neighbor_mode="on"), ao=None,
               label="1k helices x100 pts, 64^3, 256x256 opaque, neighbour on"),
    "tiny": dict(gen="turbulence", n=2000, pts=60, dims=(32, 32, 32), W=320, H=180,
                 params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed"),
                 ao=(32, 4.0, 1.0), label="smoke-sized workload"),
}


def make_lines(wl):
    from paper_1801_01155_b200 import synth
    return getattr(synth, wl["gen"])(wl["n"], wl["pts"], wl["dims"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                      "-i", str(self.index)], capture_output=True, text=True, timeout=5).stdout
                self.rows.append([c.strip() for c in out.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows if len(r) >= 6 for n, v in zip(names, r[2:6]) if v == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


# --------------------------------------------------------------------------------------
# CPU arm (oracle port of the reference): cpu_baseline and --impl reference
# --------------------------------------------------------------------------------------

def oracle_model(wl, lines):
    from oracle import lvx_oracle as orc
    pts, attrs, off = lines
    t0 = time.perf_counter()
    ref = orc.build_voxel_model(pts, attrs, off, wl["dims"], 32)
    t_vox = time.perf_counter() - t0
    t0 = time.perf_counter()
    levels = orc.build_octree(orc.compute_density_level0(ref))
    t_lod = time.perf_counter() - t0
    t_ao = None
    if wl["ao"]:
        t0 = time.perf_counter()
        ref.ao = orc.precompute_voxel_ao(ref, levels, *wl["ao"])
        t_ao = time.perf_counter() - t0
    return orc, ref, levels, dict(voxelize_s=t_vox, lod_s=t_lod, ao_bake_s=t_ao,
                                  voxelize_mseg_s=ref.segment_count / t_vox / 1e6)


def oracle_frame_ms(orc, wl, ref, levels, row_step, threads=0):
    """Times the oracle on rows 0, row_step, 2*row_step, ... and scales to the frame."""
    W, H = wl["W"], wl["H"]
    kw = dict(wl["params"])
    nb = kw.pop("neighbor_mode") != "off"
    rows = len(range(0, H, row_step))
    t0 = time.perf_counter()
    orc.render(orc.default_camera(wl["dims"], W, H), ref, levels, neighbor=nb, rows=(0, H, row_step),
               threads=threads, **kw)
    dt = time.perf_counter() - t0
    return dt * 1e3 * H / rows, dt, rows


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lines = make_lines(wl)
    orc, ref, levels, stage = oracle_model(wl, lines)
    cores = orc.num_threads()
    row_step = args.cpu_row_step
    per = []
    for _ in range(max(args.warmup, 0)):
        oracle_frame_ms(orc, wl, ref, levels, row_step * 4)
    for _ in range(args.steps):
        ms, dt, rows = oracle_frame_ms(orc, wl, ref, levels, row_step)
        per.append(ms)
    ms = float(np.mean(per))
    sample = f"rows 0::{row_step} of the {wl['W']}x{wl['H']} frame ({rows} rows), scaled by H/rows"
    line = {
        "impl": "reference", "metric": "ms_per_frame", "value": ms, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["label"], "segments": int(ref.segment_count)},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port", "sample": sample,
                         **{k: v for k, v in stage.items() if v is not None}},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": "CPU path: C port (oracle/lvx_oracle.c, OpenMP) of the Python/numba reference, pinned "
                "bit-exact to it; the reference itself cannot travel to the GPU box",
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------

def run_ours(args, wl):
    import torch
    import torch.distributed as dist
    import paper_1801_01155_b200 as lv
    from paper_1801_01155_b200 import _lib, parallel
    from paper_1801_01155_b200.illumination import ao_bake_device
    from paper_1801_01155_b200.lod import density_level0_device, _octree_from_level0_device
    from paper_1801_01155_b200.raycast import FramePlan, resolve_neighbor

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return float(x)
        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def ev_ms(fn, reps=1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    peak, peak_src = measured_peak()
    dims, W, H = wl["dims"], wl["W"], wl["H"]
    spec = lv.GridSpec(dims, 32)
    lines = make_lines(wl)
    pts, attrs, off = lines
    n_curves = int(off.size - 1)
    V = spec.voxel_count
    launches = {"n": 0}

    # ---- stages (untimed w.r.t. the headline; each timed on its own) --------------------
    stages = {}
    pts_d, attrs_d, off_d = _lib.to_device(pts), _lib.to_device(attrs), _lib.to_device(off)
    lv.voxelize_device(pts_d, attrs_d, off_d, n_curves, spec, caches=False, provenance=False)  # warm-up
    t_vox = min(ev_ms(lambda: lv.voxelize_device(pts_d, attrs_d, off_d, n_curves, spec, caches=False,
                                                 provenance=False)) for _ in range(3))
    t0 = time.perf_counter()
    model = lv.build_voxel_model(lv.CurveSet.from_flat(pts, attrs, off), spec)
    torch.cuda.synchronize()
    t_vox_e2e = (time.perf_counter() - t0) * 1e3
    S = model.segment_count
    P = int(pts.shape[0])
    b_vox = 32 * P + S * (5 + 26) + 5 * V
    stages["voxelize"] = {"ms": t_vox, "mseg_per_s": S / t_vox / 1e3, "alg_bytes": b_vox,
                          "gbs": b_vox / t_vox / 1e6, "frac_of_hbm_peak": b_vox / t_vox / 1e6 / peak,
                          "e2e_ms_host_arrays_in_model_out": t_vox_e2e, "segments": S, "vertices": P}
    l0 = density_level0_device(model)
    t_l0 = min(ev_ms(lambda: density_level0_device(model)) for _ in range(3))
    t_mip = min(ev_ms(lambda: _octree_from_level0_device(l0, dims)) for _ in range(3))
    b_lod = 25 * S + 4 * V + 4 * V * (8 / 7 + 1 / 7)
    stages["lod"] = {"ms": t_l0 + t_mip, "density_ms": t_l0, "mip_ms": t_mip, "alg_bytes": int(b_lod),
                     "gbs": b_lod / (t_l0 + t_mip) / 1e6, "frac_of_hbm_peak": b_lod / (t_l0 + t_mip) / 1e6 / peak}
    octree = lv.build_lod(model)
    if wl["ao"]:
        aop = lv.AOParams(n_rays=wl["ao"][0], radius=wl["ao"][1], step=wl["ao"][2])
        ao_bake_device(model, octree, aop)
        t_ao = min(ev_ms(lambda: ao_bake_device(model, octree, aop)) for _ in range(2))
        occupied = int((model.dev("counts") > 0).sum().item())
        samples = occupied * wl["ao"][0] * int(wl["ao"][1] / wl["ao"][2])
        stages["ao_bake"] = {"ms": t_ao, "occupied_voxels": occupied, "gsamples_per_s": samples / t_ao / 1e6,
                             "requested_gbs": samples * 32 / t_ao / 1e6}
        model.ao = lv.precompute_voxel_ao(model, octree, aop)

    # ---- the frame ---------------------------------------------------------------------------
    params = lv.RenderParams(**wl["params"])
    cam = lv.default_camera(dims, W, H)
    nb = resolve_neighbor(params, False)
    if world == 1:
        plan = FramePlan(cam, model, octree, params, nb)
        img_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    else:
        plan = FramePlan(cam, model, octree, params, nb, tile_first=rank, tile_step=world, compact=True,
                         tile_w=parallel.MG_TILE_W, tile_h=parallel.MG_TILE_H)
        img_d = torch.zeros((max(plan.n_my_tiles(), 1), parallel.MG_TILE_H, parallel.MG_TILE_W, 4),
                            dtype=torch.float32, device="cuda")
        full_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda") if rank == 0 else None
    stats_d = torch.zeros((H, 3), dtype=torch.int64, device="cuda")

    L = _lib.lib()

    def frame_launches():
        """kernels of this repo launched by the last plan.launch()"""
        return int(L.lvx_render_wf_last_launches(None)) if plan.engine == "wavefront" else 1

    def step():
        plan.launch(img_d, stats_d)
        launches["n"] += frame_launches()
        if world > 1:
            parts = parallel.gather_tiles(img_d[:plan.n_my_tiles()], 0)
            if rank == 0:
                for r, part in enumerate(parts):
                    parallel.untile_into(part, r, world, W, H, full_d)
                    launches["n"] += 1

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    stats_d.zero_()
    n0 = launches["n"]
    kern_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record()
        for i in range(args.steps):
            kern_ev[i][0].record()
            plan.launch(img_d, stats_d)
            kern_ev[i][1].record()
            launches["n"] += frame_launches()
            if world > 1:
                parts = parallel.gather_tiles(img_d[:plan.n_my_tiles()], 0)
                if rank == 0:
                    for r, part in enumerate(parts):
                        parallel.untile_into(part, r, world, W, H, full_d)
                        launches["n"] += 1
        e1.record()
        barrier()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    ms_frame = total_ms / args.steps
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in kern_ev]))
    gpu_launches = launches["n"] - n0
    tot = (stats_d.sum(0) // args.steps)
    if world > 1:
        dist.all_reduce(tot)
    tot = tot.tolist()

    # ---- e2e through the public API ---------------------------------------------------------
    def api_frame():
        if world == 1:
            return lv.render_frame(cam, model, octree, None, params)
        return parallel.render_frame_tiled(cam, model, octree, None, params)

    for _ in range(2):
        api_frame()
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fr = api_frame()
    barrier()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / args.steps)
    h2d = ctypes.sizeof(_lib.Camera) + ctypes.sizeof(_lib.Params) + ctypes.sizeof(_lib.Model) + \
        ctypes.sizeof(_lib.Lod) + ctypes.sizeof(_lib.Tiling)
    d2h = W * H * 16 + 24

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the frame kernel (rank 0, single GPU view) -----------------------------
    bits = torch.zeros((V + 31) // 32, dtype=torch.int32, device="cuda")
    plan1 = FramePlan(cam, model, octree, params, nb)
    img1 = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    st1 = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
    plan1.launch_footprint(img1, st1, bits)
    torch.cuda.synchronize()
    b8 = bits.view(torch.uint8)
    touched = torch.stack([(b8 >> k) & 1 for k in range(8)], dim=1).reshape(-1)[:V].bool()
    n_vox = int(touched.sum().item())
    n_seg = int(model.dev("counts")[touched].sum(dtype=torch.int64).item())
    alg_bytes = 6 * n_vox + 32 * n_seg + 16 * W * H
    lit = float((img1[..., :3].sum(-1) > 0).float().mean().item())
    tot1 = st1.sum(0).tolist()
    requested = tot1[0] + 32 * (tot1[1] // (3 if params.joint_spheres else 1)) + 16 * W * H
    k1 = kern_ms if world == 1 else min(ev_ms(lambda: plan1.launch(img1, st1)) for _ in range(2))
    kname = "render_kernel" if plan.engine == "tile" else \
        "wavefront frame: wf_init + N x (wf_walk, wf_cand, wf_exact<tube>, wf_exact<sphere>, wf_composite)"
    roofline = {"bound": "hbm", "kernel": kname, "engine": plan.engine, "achieved": alg_bytes / k1 / 1e6, "peak": peak,
                "unit": "GB/s", "frac": alg_bytes / k1 / 1e6 / peak, "traffic": None,
                "peak_source": peak_src, "alg_bytes_per_launch": alg_bytes, "voxels_touched": n_vox,
                "segments_touched": n_seg, "kernel_ms": k1, "requested_bytes": requested,
                "requested_gbs": requested / k1 / 1e6,
                "note": "unique bytes the reference's algorithm touches per frame (6 B/voxel header+occupancy, "
                        "32 B/segment, 16 B/pixel out); the frame is latency / L2-transaction bound, not HBM bound "
                        "(see profiles/); kernel_ms is the CUDA-event time of the whole frame"}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            roofline["traffic"] = json.load(open(prof)).get(args.workload, {}).get(
                "render_kernel" if plan.engine == "tile" else "wavefront_frame")
        except Exception:
            pass

    # ---- cpu baseline (bounded sample, rank 0, N == 1 only) -----------------------------------
    cpu = None
    if world == 1 and not args.no_cpu:
        orc, ref, levels, stage_cpu = oracle_model(wl, lines)
        ms_cpu, dt, rows = oracle_frame_ms(orc, wl, ref, levels, args.cpu_row_step)
        cpu = {"value": ms_cpu, "unit": "ms", "cores": orc.num_threads(), "kind": "port",
               "sample": f"rows 0::{args.cpu_row_step} of the same {W}x{H} frame ({rows} rows, {dt:.1f} s), "
                         "scaled by H/rows; voxelize/LoD/AO timed in full",
               **{k: v for k, v in stage_cpu.items() if v is not None}}

    line = {
        "metric": "ms_per_frame", "value": ms_frame, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_frame, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["label"], "segments": S, "voxels": V, "bins": 32, "camera": "default_camera",
                   "lit_pixel_fraction": lit, "rays_per_s": W * H / ms_frame * 1e3,
                   "l2": "no flush: the model (%.0f MB of records+headers+AO) exceeds the 126 MB L2" %
                         ((32 * S + 5 * V + 4 * V + (dims[0] + 2) * (dims[1] + 2) * (dims[2] + 2)) / 1e6),
                   "parallelism": "1 GPU" if world == 1 else f"{world} GPUs, interleaved {parallel.MG_TILE_W}x"
                                  f"{parallel.MG_TILE_H} screen tiles, NCCL gather to rank 0"},
        "frame_stats": {"voxel_steps": tot[0], "intersection_tests": tot[1], "window_overflow": tot[2]},
        "kernel_ms": kern_ms, "engine": plan.engine,
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "render_frame" if world == 1 else "render_frame_tiled",
                "image_path": ("kernels write each finished pixel into the pinned host image through its device "
                               "mapping (counted in d2h_bytes_per_step); counters copied after the frame")
                if world == 1 else "tiles gathered to rank 0 over NCCL, then one copy to pinned host memory"},
        "gpu_launches": gpu_launches,
        "clocks": clocks.summary(),
        "roofline": roofline,
        "stages": stages,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--cpu-row-step", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
