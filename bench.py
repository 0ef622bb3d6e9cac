#!/usr/bin/env python
"""bench.py -- ms/frame of the linevox hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c2|c1|c4_1080p|c4|c5|tiny] [--no-cpu] [--no-targets]

Default workload (BASELINE.json configs[2], the config the metric "transparent+AO, 1080p"
is quoted on): 100k turbulence-like synthetic lines x 100 points, 256^3 grid,
N=32 bins -> 9.68 M segments; 1920x1080, alpha = 0.25, tau = 0.95, neighbour mode
on, precomputed LoD ambient occlusion (100 rays, radius 5).  A "step" is one frame.

* `value`    device time per frame (CUDA events around K frames, inputs resident in HBM).
* `e2e`      the same frame through the public API `render_frame` (`render_frame_tiled`
             for N > 1): camera/params from host objects, image copied back to pinned
             host memory and the counters read every step.
* `parity`   the GPU frame against the rows the CPU oracle renders for `cpu_baseline`
             (max / mean per-channel error, per-row counters equal).
* `roofline` the frame kernel against the measured HBM peak, from the unique bytes the
             reference's algorithm touches (instrumented pass).
* `stages`   voxelize / LoD / AO bake timings of the same data set (Mseg/s, GB/s).
* `variants` the same scene in own-voxel mode, with density-ray AO and with cone shadows
             (SURVEY.md 8d asks for them; the reference's bench loop is cli.py:255-290).
* `targets`  the north_star target configurations, measured in the same run: the 1 M-line /
             256^3 set (BASELINE configs[3]'s scene) voxelized (C5's first point) and rendered at
             1080p (<= 16 ms target) and at 4K with cone shadows, each with its own clock sample.
* `cpu_baseline` the CPU oracle (a C port of the reference, OpenMP) on every 2nd row of the
             same frame.

Other workloads: `c4_1080p` / `c4` put the 1 M-line scene in the headline; `c5` is the
voxelization-only sweep point (metric Mseg/s; N > 1 shards the lines by ID and all-gathers).
N > 1: launched by torchrun -- or by this script itself when WORLD_SIZE is not set; the image is
split into interleaved tiles (strong scaling).  `--impl reference` times the CPU path only (the
Python/numba reference cannot travel to the GPU box; the pinned C port stands in).
"""
import argparse
import ctypes
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

AO_BAKE = (100, 5.0, 1.0)
WORKLOADS = {
    # name: generator, n_lines, pts, dims, W, H, RenderParams kwargs, AO bake
    "c3": dict(gen="turbulence", n=100000, pts=100, dims=(256, 256, 256), W=1920, H=1080,
               params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed"),
               ao=AO_BAKE,
               label="100k turbulence lines x100 pts, 256^3, 1080p transparent(alpha .25)+precomputed AO, neighbour on"),
    "c2": dict(gen="helices", n=10000, pts=100, dims=(128, 128, 128), W=1920, H=1080,
               params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on"), ao=None,
               label="10k helices x100 pts, 128^3, 1080p transparent(alpha .25), neighbour on"),
    "c1": dict(gen="helices", n=1000, pts=100, dims=(64, 64, 64), W=256, H=256,
               params=dict(neighbor_mode="on"), ao=None,
               label="1k helices x100 pts, 64^3, 256x256 opaque, neighbour on"),
    # BASELINE configs[3]'s scene on one GPU at 1080p: the north_star "<= 16 ms" target
    "c4_1080p": dict(gen="turbulence", n=1000000, pts=100, dims=(256, 256, 256), W=1920, H=1080,
                     params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed"),
                     ao=AO_BAKE,
                     label="1M turbulence lines x100 pts, 256^3, 1080p transparent(alpha .25)+precomputed AO, neighbour on"),
    # BASELINE configs[3]: 4K, transparent + AO + soft (cone) shadows
    "c4": dict(gen="turbulence", n=1000000, pts=100, dims=(256, 256, 256), W=3840, H=2160,
               params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed",
                           shadow_mode="cone", light_dir=(0.3, 0.2, 1.0)),
               ao=AO_BAKE,
               label="1M turbulence lines x100 pts, 256^3, 4K transparent(alpha .25)+precomputed AO+cone shadows, neighbour on"),
    # BASELINE configs[4]: voxelization only (first point of the 1M-10M sweep; --lines for the others)
    "c5": dict(gen="turbulence", n=1000000, pts=100, dims=(256, 256, 256), W=0, H=0, params=None, ao=None,
               voxelize_only=True, label="voxelization only: {n} turbulence lines x100 pts, 256^3, N=32"),
    "tiny": dict(gen="turbulence", n=2000, pts=60, dims=(32, 32, 32), W=320, H=180,
                 params=dict(base_opacity=0.25, tau=0.95, neighbor_mode="on", ao_mode="precomputed"),
                 ao=(32, 4.0, 1.0), label="smoke-sized workload"),
}

# `variants` of the headline scene
VARIANTS = (
    ("own_voxel", dict(neighbor_mode="off"), "neighbour off (the paper's interactive mode)"),
    ("density_rays_ao", dict(ao_mode="density-rays", ao_rays=25, ao_radius=15.0), "AO by 25 density rays per hit, R=15"),
    ("cone_shadows", dict(shadow_mode="cone", light_dir=(0.3, 0.2, 1.0)), "+ cone soft shadows"),
)


def config_of(wl, S, world):
    """The `config` object both arms print (same keys and values for the same workload and N)."""
    dims = wl["dims"]
    V = dims[0] * dims[1] * dims[2]
    return {"workload": wl["label"], "segments": int(S), "voxels": V, "bins": 32, "camera": "default_camera",
            "l2": "no flush: the model (%.0f MB of records+headers+AO) exceeds the 126 MB L2" %
                  ((32 * S + 5 * V + 4 * V + (dims[0] + 2) * (dims[1] + 2) * (dims[2] + 2)) / 1e6),
            "parallelism": "1 GPU" if world == 1 else f"{world} GPUs, interleaved 32x16 screen tiles, "
                                                      "one NCCL gather to rank 0 per frame"}


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

def oracle_model(wl, lines, want_lod=True):
    from oracle import lvx_oracle as orc
    pts, attrs, off = lines
    t0 = time.perf_counter()
    ref = orc.build_voxel_model(pts, attrs, off, wl["dims"], 32)
    t_vox = time.perf_counter() - t0
    levels, t_lod, t_ao = None, None, None
    if want_lod:
        t0 = time.perf_counter()
        levels = orc.build_octree(orc.compute_density_level0(ref))
        t_lod = time.perf_counter() - t0
        if wl["ao"]:
            t0 = time.perf_counter()
            ref.ao = orc.precompute_voxel_ao(ref, levels, *wl["ao"])
            t_ao = time.perf_counter() - t0
    return orc, ref, levels, dict(voxelize_s=t_vox, lod_s=t_lod, ao_bake_s=t_ao,
                                  voxelize_mseg_s=ref.segment_count / t_vox / 1e6)


def oracle_frame(orc, wl, ref, levels, row_step, threads=0):
    """The oracle on rows 0, row_step, 2*row_step, ...: (ms scaled to the frame, seconds, rows,
    image, stats of those rows)."""
    W, H = wl["W"], wl["H"]
    kw = dict(wl["params"])
    nb = kw.pop("neighbor_mode") != "off"
    rows = len(range(0, H, row_step))
    t0 = time.perf_counter()
    img, st = orc.render(orc.default_camera(wl["dims"], W, H), ref, levels, neighbor=nb, rows=(0, H, row_step),
                         threads=threads, **kw)
    dt = time.perf_counter() - t0
    return dt * 1e3 * H / rows, dt, rows, img, st


def run_reference(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lines = make_lines(wl)
    if wl.get("voxelize_only"):
        # the numpy voxelizer of the reference is single-threaded; the port is too
        orc, ref, _, stage = oracle_model(wl, lines, want_lod=False)
        per = [stage["voxelize_mseg_s"]]
        for _ in range(max(args.steps - 1, 0)):
            per.append(oracle_model(wl, lines, want_lod=False)[3]["voxelize_mseg_s"])
        v = float(np.median(per))
        line = {
            "impl": "reference", "metric": "voxelize_mseg_per_s", "value": v, "unit": "Mseg/s", "n_gpus": args.gpus,
            "steps": len(per), "warmup": 0, "ms_per_step": ref.segment_count / v / 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl["label"].format(n=wl["n"]), "segments": int(ref.segment_count)},
            "cpu_baseline": {"value": v, "unit": "Mseg/s", "cores": 1, "kind": "port",
                             "sample": f"the whole set, {len(per)} pass(es)", "range": [min(per), max(per)]},
            "e2e": {"value": v, "unit": "Mseg/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
            "note": "CPU path: C port (oracle/lvx_oracle.c) of the reference's numpy voxelizer, pinned bit-exact to it",
        }
        print(json.dumps(line), flush=True)
        return
    orc, ref, levels, stage = oracle_model(wl, lines)
    cores = orc.num_threads()
    row_step = args.cpu_row_step
    per = []
    for _ in range(max(args.warmup, 0)):
        oracle_frame(orc, wl, ref, levels, row_step * 4)
    for _ in range(args.steps):
        ms, dt, rows, _, _ = oracle_frame(orc, wl, ref, levels, row_step)
        per.append(ms)
    ms = float(np.mean(per))
    sample = f"rows 0::{row_step} of the {wl['W']}x{wl['H']} frame ({rows} rows), scaled by H/rows"
    line = {
        "impl": "reference", "metric": "ms_per_frame", "value": ms, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(wl, ref.segment_count, args.gpus),
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port", "sample": sample,
                         "range": [float(min(per)), float(max(per))],
                         **{k: v for k, v in stage.items() if v is not None}},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
        "note": "CPU path: C port (oracle/lvx_oracle.c, OpenMP) of the Python/numba reference, pinned "
                "bit-exact to it; the reference itself cannot travel to the GPU box; run-to-run spread of "
                "this arm is about 10 % (see cpu_baseline.range)",
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------------------

class Dist:
    """Rank bookkeeping + the two collectives the timing protocol needs."""

    def __init__(self, args):
        import torch
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(self.local)
        # LVX_DIST_BACKEND=gloo: several ranks may share one GPU (collectives staged through the host);
        # only for exercising the N > 1 code path where a single GPU is all there is
        self.backend = os.environ.get("LVX_DIST_BACKEND", "nccl")
        if self.world > 1:
            import torch.distributed as dist
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            else:
                dist.init_process_group(self.backend)
        if self.world != args.gpus and self.rank == 0:
            print(f"warning: --gpus {args.gpus} but WORLD_SIZE={self.world}", file=sys.stderr)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()
        self.torch.cuda.synchronize()

    def max_over_ranks(self, x):
        if self.world == 1:
            return float(x)
        import torch.distributed as dist
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device="cuda" if self.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


def ev_ms(fn, reps=1):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def voxelize_stage(lv, lines, spec, peak, e2e_reps=2):
    """Kernel-only and end-to-end timing of the voxelizer on one line set.
    Returns (model, stage dict)."""
    import torch
    from paper_1801_01155_b200 import _lib
    pts, attrs, off = lines
    n_curves = int(off.size - 1)
    V = spec.voxel_count
    pts_d, attrs_d, off_d = _lib.to_device(pts), _lib.to_device(attrs), _lib.to_device(off)
    lv.voxelize_device(pts_d, attrs_d, off_d, n_curves, spec, caches=False, provenance=False)  # warm-up
    t_vox = min(ev_ms(lambda: lv.voxelize_device(pts_d, attrs_d, off_d, n_curves, spec, caches=False,
                                                 provenance=False)) for _ in range(3))
    del pts_d, attrs_d, off_d
    cs = lv.CurveSet.from_flat(pts, attrs, off)
    e2e = []
    model = None
    for _ in range(e2e_reps):
        model = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        model = lv.build_voxel_model(cs, spec)
        torch.cuda.synchronize()
        e2e.append((time.perf_counter() - t0) * 1e3)
    S = model.segment_count
    P = int(pts.shape[0])
    b_vox = 32 * P + S * (5 + 26) + 5 * V
    h2d = pts.nbytes + attrs.nbytes + off.nbytes
    st = {"ms": t_vox, "mseg_per_s": S / t_vox / 1e3, "alg_bytes": b_vox, "gbs": b_vox / t_vox / 1e6,
          "frac_of_hbm_peak": b_vox / t_vox / 1e6 / peak,
          "e2e_ms": min(e2e), "e2e_ms_first_call": e2e[0], "e2e_mseg_per_s": S / min(e2e) / 1e3,
          "e2e_bytes": {"h2d_vertices": int(h2d), "d2h": 24,
                        "note": "build_voxel_model(CurveSet of host arrays) -> VoxelModel whose arrays stay on the "
                                "device until read; the host copy of the vertices is the bulk of the time"},
          "segments": S, "vertices": P}
    return model, st


def time_frame(plan, img_d, stats_d, steps, warmup=3):
    for _ in range(warmup):
        plan.launch(img_d, stats_d)
    return ev_ms(lambda: plan.launch(img_d, stats_d), steps)


def run_voxelize_only(args, wl, D):
    """C5: voxelization-only.  value = segments / time, inputs resident in HBM; N > 1: lines sharded by
    ID, per-voxel counts all-reduced and raw records all-gathered, every rank builds the full model."""
    import torch
    import paper_1801_01155_b200 as lv
    from paper_1801_01155_b200 import _lib, parallel, voxelizer as vz
    peak, peak_src = measured_peak()
    spec = lv.GridSpec(wl["dims"], 32)
    lines = make_lines(wl)
    pts, attrs, off = lines
    n_curves = int(off.size - 1)
    P = int(pts.shape[0])
    world, rank = D.world, D.rank
    launches_per = 9  # mark, bound, clip, 3 x scan, regroup, compact (+ memsets); provenance off
    if world == 1:
        pts_d, attrs_d, off_d = _lib.to_device(pts), _lib.to_device(attrs), _lib.to_device(off)

        def step():
            return lv.voxelize_device(pts_d, attrs_d, off_d, n_curves, spec, caches=False, provenance=False)
    else:
        import torch.distributed as dist
        c0, c1 = parallel.shard_range(n_curves, rank, world)
        p0, p1 = int(off[c0]), int(off[c1])
        pts_d, attrs_d = _lib.to_device(pts[p0:p1]), _lib.to_device(attrs[p0:p1])
        off_d = _lib.to_device(off[c0:c1 + 1] - p0)

        def step():
            sh = parallel.voxelize_shard(pts_d, attrs_d, off_d, c1 - c0, spec, p0, want_edge_kept=False)
            total = parallel.all_reduce_(sh["vox_cnt"].clone())
            keys, qs, lins = parallel.allgather_varlen_multi([sh["raw_key"], sh["raw_q"], sh["raw_lin"]])
            return parallel.merge_shards(spec, total, torch.cat(keys), torch.cat(qs), torch.cat(lins), caches=False)
    for _ in range(max(args.warmup, 3)):
        out = step()
    S = int(out["n_segments"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(D.local) as clocks:
        D.barrier()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        D.barrier()
    ms = D.max_over_ranks(e0.elapsed_time(e1)) / args.steps
    del out
    # e2e: the public API with host arrays in, the model's packed bytes resident on the device out
    cs = lv.CurveSet.from_flat(pts, attrs, off)
    api = (lambda: lv.build_voxel_model(cs, spec)) if world == 1 else (lambda: parallel.build_voxel_model_sharded(cs, spec))
    api()
    D.barrier()
    t0 = time.perf_counter()
    n_e2e = max(1, min(args.steps, 3))
    for _ in range(n_e2e):
        api()
    D.barrier()
    e2e_ms = D.max_over_ranks((time.perf_counter() - t0) * 1e3 / n_e2e)
    if rank != 0:
        D.close()
        return
    V = spec.voxel_count
    b_vox = 32 * P + S * (5 + 26) + 5 * V
    cpu = None
    if world == 1 and not args.no_cpu:
        # bounded sample: the first 100k lines of the same set (the port is single-threaded like numpy)
        n_s = min(100000, n_curves)
        sub = (pts[:off[n_s]], attrs[:off[n_s]], off[:n_s + 1])
        orc, ref, _, st = oracle_model(dict(wl, n=n_s), sub, want_lod=False)
        cpu = {"value": st["voxelize_mseg_s"], "unit": "Mseg/s", "cores": 1, "kind": "port",
               "sample": f"the first {n_s} lines of the same set ({ref.segment_count} segments, {st['voxelize_s']:.1f} s)"}
    line = {
        "metric": "voxelize_mseg_per_s", "value": S / ms / 1e3, "unit": "Mseg/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["label"].format(n=wl["n"]), "segments": S, "vertices": P, "voxels": V, "bins": 32,
                   "l2": "no flush: vertices + records (%.1f GB) exceed the 126 MB L2" % (b_vox / 1e9),
                   "parallelism": "1 GPU" if world == 1 else f"{world} GPUs, lines sharded by ID, all-reduce of "
                                  "per-voxel counts + all-gather of raw records, replicated model",
                   **({"backend": D.backend + " (ranks share GPUs: a code-path exercise, not a scaling number)"}
                      if D.backend != "nccl" else {})},
        "e2e": {"value": S / e2e_ms / 1e3, "unit": "Mseg/s", "ms": e2e_ms, "h2d_bytes_per_step": int(pts.nbytes + attrs.nbytes + off.nbytes),
                "d2h_bytes_per_step": 24, "api": "build_voxel_model" if world == 1 else "build_voxel_model_sharded"},
        "gpu_launches": launches_per * args.steps,
        "clocks": clocks.summary(),
        "roofline": {"bound": "hbm", "kernel": "voxelizer pipeline (clip + scan + regroup + compact)", "achieved": b_vox / ms / 1e6,
                     "peak": peak, "unit": "GB/s", "frac": b_vox / ms / 1e6 / peak, "traffic": None, "peak_source": peak_src,
                     "alg_bytes_per_launch": b_vox},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    D.close()


def run_ours(args, wl):
    import torch
    import paper_1801_01155_b200 as lv
    from paper_1801_01155_b200 import _lib, parallel
    from paper_1801_01155_b200.illumination import ao_bake_device
    from paper_1801_01155_b200.lod import density_level0_device, mips_inplace, octree_buffer
    from paper_1801_01155_b200.raycast import FramePlan, resolve_neighbor

    D = Dist(args)
    if wl.get("voxelize_only"):
        return run_voxelize_only(args, wl, D)
    world, rank, local = D.world, D.rank, D.local
    barrier, max_over_ranks = D.barrier, D.max_over_ranks

    peak, peak_src = measured_peak()
    dims, W, H = wl["dims"], wl["W"], wl["H"]
    spec = lv.GridSpec(dims, 32)
    lines = make_lines(wl)
    V = spec.voxel_count
    launches = {"n": 0}

    # ---- stages (untimed w.r.t. the headline; each timed on its own) --------------------
    stages = {}
    model, stages["voxelize"] = voxelize_stage(lv, lines, spec, peak)
    S = model.segment_count

    def lod_and_ao(model, ao):
        st = {}
        flat, v0 = octree_buffer(dims)
        density_level0_device(model, out=flat[:v0])
        t_l0 = min(ev_ms(lambda: density_level0_device(model, out=flat[:v0])) for _ in range(3))
        t_mip = min(ev_ms(lambda: mips_inplace(flat, dims)) for _ in range(3))
        del flat
        Sm = model.segment_count
        b_lod = 25 * Sm + 4 * V + 4 * V * (8 / 7 + 1 / 7)
        st["lod"] = {"ms": t_l0 + t_mip, "density_ms": t_l0, "mip_ms": t_mip, "alg_bytes": int(b_lod),
                     "gbs": b_lod / (t_l0 + t_mip) / 1e6, "frac_of_hbm_peak": b_lod / (t_l0 + t_mip) / 1e6 / peak}
        octree = lv.build_lod(model)
        if ao:
            aop = lv.AOParams(n_rays=ao[0], radius=ao[1], step=ao[2])
            ao_bake_device(model, octree, aop)
            t_ao = min(ev_ms(lambda: ao_bake_device(model, octree, aop)) for _ in range(2))
            occupied = int((model.dev("counts") > 0).sum().item())
            samples = occupied * ao[0] * int(ao[1] / ao[2])
            # bound: the FP64 pipe (cache-resident, no FMA): ~58 float64-pipe instructions per trilinear
            # sample in the interior path (SASS count); peak = SMs x 64 lanes x clock
            fp64_peak = 148 * 64 * 1.965e9
            st["ao_bake"] = {"ms": t_ao, "occupied_voxels": occupied, "gsamples_per_s": samples / t_ao / 1e6,
                             "samples_upper_bound": samples, "requested_gbs": samples * 32 / t_ao / 1e6,
                             "bound": "fp64 pipe", "fp64_ops_per_sample": 58,
                             "frac_of_fp64_pipe_peak_upper_bound": samples * 58 / (t_ao * 1e-3) / fp64_peak,
                             "note": "samples = occupied x rays x floor(R/step) is an upper bound (rays stop at "
                                     "saturation or the grid border); ncu: sm__inst_executed_pipe_fp64 53 % "
                                     "(profiles/r2q_stage_kernels.txt)"}
            model.ao = lv.precompute_voxel_ao(model, octree, aop)
        return octree, st

    octree, st = lod_and_ao(model, wl["ao"])
    stages.update(st)

    # ---- the frame ---------------------------------------------------------------------------
    params = lv.RenderParams(**wl["params"])
    cam = lv.default_camera(dims, W, H)
    nb = resolve_neighbor(params, False)
    if world == 1:
        plan = FramePlan(cam, model, octree, params, nb)
        img_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
        send = recv = full_d = None
    else:
        plan = FramePlan(cam, model, octree, params, nb, tile_first=rank, tile_step=world, compact=True,
                         tile_w=parallel.MG_TILE_W, tile_h=parallel.MG_TILE_H)
        # the kernels render straight into the front of the send buffer; its tail carries the counters
        send = parallel.new_send_buffer(world, W, H, "cuda")
        img_d = parallel.send_tiles_view(send, max(plan.n_my_tiles(), 1))
        full_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda") if rank == 0 else None
        recv = torch.empty((world, send.numel()), dtype=torch.float32, device="cuda") if rank == 0 else None
    stats_d = torch.zeros((H, 3), dtype=torch.int64, device="cuda")

    L = _lib.lib()

    def frame_launches():
        """kernels of this repo launched by the last plan.launch()"""
        return int(L.lvx_render_wf_last_launches(None)) if plan.engine == "wavefront" else 1

    def step():
        plan.launch(img_d, stats_d)
        launches["n"] += frame_launches()
        if world > 1:
            parallel.pack_counters(send, stats_d.sum(dim=0))
            parallel.gather_tiles(send, 0, recv=recv)   # ONE collective per frame
            if rank == 0:
                parallel.untile_all(recv, world, W, H, full_d)
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
                parallel.pack_counters(send, stats_d.sum(dim=0))
                parallel.gather_tiles(send, 0, recv=recv)
                if rank == 0:
                    parallel.untile_all(recv, world, W, H, full_d)
                    launches["n"] += 1
        e1.record()
        barrier()
    total_ms = max_over_ranks(e0.elapsed_time(e1))
    ms_frame = total_ms / args.steps
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in kern_ev]))
    gpu_launches = launches["n"] - n0
    row_tot = (stats_d // args.steps)
    if world > 1:
        parallel.all_reduce_(row_tot)
    gpu_row_stats = row_tot.cpu().numpy()
    tot = gpu_row_stats.sum(0).tolist()

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
        D.close()
        return
    engine = plan.engine
    gpu_image = np.array(fr.image, copy=True)   # the frame the public API returned (host memory)

    # ---- roofline of the frame kernel (rank 0, single GPU view) -----------------------------
    bits = torch.zeros((V + 31) // 32, dtype=torch.int32, device="cuda")
    plan1 = FramePlan(cam, model, octree, params, nb, records="rec")
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
    del bits, b8, touched
    k1 = kern_ms if world == 1 else min(ev_ms(lambda: plan1.launch(img1, st1)) for _ in range(2))
    kname = "render_kernel" if plan.engine == "tile" else \
        "wavefront frame: wf_init + N x (wf_walk, wf_cand, wf_exact, wf_composite, wf_next)"
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

    # ---- variants of the same scene (rank 0, one GPU) ---------------------------------------
    variants = {}
    if world == 1 and not args.no_variants:
        for name, extra, what in VARIANTS:
            kw = dict(wl["params"])
            kw.update(extra)
            pv = lv.RenderParams(**kw)
            planv = FramePlan(cam, model, octree, pv, resolve_neighbor(pv, False))
            stv = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
            with ClockSampler(local) as ck:
                msv = time_frame(planv, img1, stv, max(3, min(args.steps, 10)))
            variants[name] = {"ms": msv, "engine": planv.engine, "what": what, "clocks": ck.summary()}

    # ---- cpu baseline + parity (bounded sample, rank 0, N == 1 only) ---------------------------
    cpu = parity = None
    if world == 1 and not args.no_cpu:
        orc, ref, levels, stage_cpu = oracle_model(wl, lines)
        per = []
        for _ in range(2):
            ms_cpu, dt, rows, cpu_img, cpu_st = oracle_frame(orc, wl, ref, levels, args.cpu_row_step)
            per.append(ms_cpu)
        cpu = {"value": float(np.mean(per)), "unit": "ms", "cores": orc.num_threads(), "kind": "port",
               "range": [float(min(per)), float(max(per))],
               "sample": f"rows 0::{args.cpu_row_step} of the same {W}x{H} frame ({rows} rows, {dt:.1f} s), "
                         "scaled by H/rows, 2 passes; voxelize/LoD/AO timed in full",
               **{k: v for k, v in stage_cpu.items() if v is not None}}
        # parity of the frame that was timed: the oracle's rows against the same rows of the GPU image
        sel = np.arange(0, H, args.cpu_row_step)
        err = np.abs(gpu_image[sel].astype(np.float64) - cpu_img[sel].astype(np.float64))
        sub = gpu_row_stats[sel].sum(0).tolist()
        parity = {"rows": int(sel.size), "row_step": args.cpu_row_step, "max_err": float(err.max()),
                  "mean_err": float(err.mean()), "pixels_differing": int((err.max(-1) > 0).sum()),
                  "bar": "max <= 1/255 and mean < 1e-3 (north_star)",
                  "ok": bool(err.max() <= 1.0 / 255.0 and err.mean() < 1e-3),
                  "counters_equal": bool(sub[0] == cpu_st["voxel_steps"] and sub[1] == cpu_st["intersection_tests"]
                                         and sub[2] == cpu_st["window_overflow"]),
                  "counters_gpu_rows": sub,
                  "counters_oracle_rows": [cpu_st["voxel_steps"], cpu_st["intersection_tests"], cpu_st["window_overflow"]],
                  "model_equal": bool(np.array_equal(model.packed, ref.packed) and np.array_equal(model.counts, ref.counts)),
                  "ao_equal": (bool(np.array_equal(np.asarray(model.ao), np.asarray(ref.ao))) if wl["ao"] else None)}
        del orc, ref, levels, cpu_img

    # ---- north_star targets, measured in this run (rank 0, N == 1, default workload) -----------
    targets = None
    if world == 1 and args.workload == "c3" and not args.no_targets:
        del plan, plan1, model, octree, img_d, img1
        torch.cuda.empty_cache()
        targets = run_targets(lv, local, peak, lod_and_ao)

    line = {
        "metric": "ms_per_frame", "value": ms_frame, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_frame, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(wl, S, world),
        "lit_pixel_fraction": lit, "rays_per_s": W * H / ms_frame * 1e3,
        "frame_stats": {"voxel_steps": tot[0], "intersection_tests": tot[1], "window_overflow": tot[2]},
        "kernel_ms": kern_ms, "engine": engine,
        "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "render_frame" if world == 1 else "render_frame_tiled",
                "image_path": ("kernels write each finished pixel into the pinned host image through its device "
                               "mapping (counted in d2h_bytes_per_step); counters copied after the frame")
                if world == 1 else "tiles + counters gathered to rank 0 with one NCCL gather, one untile launch, "
                                   "then one copy to pinned host memory"},
        "gpu_launches": gpu_launches,
        "clocks": clocks.summary(),
        "roofline": roofline,
        "stages": stages,
    }
    if D.backend != "nccl":
        line["backend"] = D.backend + ": ranks share GPUs, collectives staged through the host -- a code-path exercise, not a scaling number"
    if parity:
        line["parity"] = parity
    if variants:
        line["variants"] = variants
    if targets:
        line["targets"] = targets
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    D.close()


def run_targets(lv, local, peak, lod_and_ao):
    """The 1 M-line scene of BASELINE configs[3] on this one GPU: voxelization (C5's first sweep
    point) and the frames north_star sets targets on.  Every figure has its own clock sample."""
    import torch
    from paper_1801_01155_b200.raycast import FramePlan, resolve_neighbor
    wl = WORKLOADS["c4_1080p"]
    dims = wl["dims"]
    spec = lv.GridSpec(dims, 32)
    t0 = time.perf_counter()
    lines = make_lines(wl)
    gen_s = time.perf_counter() - t0
    out = {"scene": "1M turbulence lines x100 pts, 256^3 (BASELINE configs[3] / configs[4] first point)",
           "generate_s": gen_s}
    with ClockSampler(local) as ck:
        model, vs = voxelize_stage(lv, lines, spec, peak, e2e_reps=2)  # (first call: fresh device allocations)
    vs["clocks"] = ck.summary()
    out["voxelize_1m_lines"] = vs
    del lines
    octree, st = lod_and_ao(model, wl["ao"])
    out["lod_1m_lines"] = st["lod"]
    out["ao_bake_1m_lines"] = st["ao_bake"]
    frames = (("frame_1080p_alpha_ao", 1920, 1080, wl["params"], "north_star target: <= 16 ms on 1 GPU"),
              ("frame_1080p_own_voxel", 1920, 1080, dict(wl["params"], neighbor_mode="off"), "neighbour off"),
              ("frame_4k_alpha_ao_cone", 3840, 2160, WORKLOADS["c4"]["params"], "BASELINE configs[3] frame on ONE GPU"))
    for name, W, H, kw, what in frames:
        p = lv.RenderParams(**kw)
        cam = lv.default_camera(dims, W, H)
        plan = FramePlan(cam, model, octree, p, resolve_neighbor(p, False))
        img = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
        stt = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
        with ClockSampler(local) as ck:
            ms = time_frame(plan, img, stt, 10)
        stt.zero_()
        plan.launch(img, stt)
        tt = stt.sum(0).tolist()
        out[name] = {"ms": ms, "engine": plan.engine, "what": what, "rays_per_s": W * H / ms * 1e3,
                     "frame_stats": {"voxel_steps": tt[0], "intersection_tests": tt[1], "window_overflow": tt[2]},
                     "clocks": ck.summary()}
        del plan, img
    return out


def self_launch(args):
    """`python bench.py --gpus N` without torchrun: start the N ranks ourselves."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ)
    # rank 0 prints NCCL's communicator lines (N ranks, NVLS / P2P transport) to stderr
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd, env=env))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--lines", type=int, default=0, help="c5: number of lines (default 1M)")
    ap.add_argument("--cpu-row-step", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-targets", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    args = ap.parse_args()
    wl = dict(WORKLOADS[args.workload])
    if args.lines > 0:
        wl["n"] = args.lines
    if wl.get("voxelize_only") and args.steps == 100:
        args.steps = 10
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
