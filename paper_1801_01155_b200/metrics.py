"""Reference renderer and small accounting helpers (metrics.py:58-160 of the reference).

`brute_force_render` tests every primitive at every pixel on the GPU (lvx_brute_count /
lvx_brute_render): no DDA, no windows, no ownership -- only the primitive tests, the
shading terms and the compositing rules are shared with `render_frame`, so the two
agreeing to the bit is evidence about traversal and gathering (the reference uses its own
brute-force renderer the same way, tests/test_metrics.py:117-125)."""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np

from . import _lib
from .raycast import Camera, Frame, FramePlan, RenderParams

__all__ = ["brute_force_render", "image_compare", "memory_report"]

MAX_PIXEL_HITS = 8192  # _kernels.py:37


def brute_force_render(camera: Camera, model, octree=None, replines=None, params: Optional[RenderParams] = None,
                       workers: int = 1) -> Frame:
    """Render by testing all primitives at every pixel (metrics.py:58-107).  Meant for small
    scenes: the work is pixels x segments."""
    if params is None:
        params = RenderParams()
    torch = _lib.require_device()
    L, st = _lib.lib(), _lib.stream_ptr()
    plan = FramePlan(camera, model, octree, params, 0, engine="tile", replines=replines)
    H, W = int(camera.height), int(camera.width)
    S = int(model.segment_count)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    count = torch.zeros(W * H, dtype=torch.int32, device="cuda")
    _lib.check(L.lvx_brute_count(C.byref(plan.cam), C.byref(plan.mdl), C.byref(plan.par), C.c_int64(S),
                                 _lib.ptr(count), st))
    kept = count.to(torch.int64).clamp_(max=MAX_PIXEL_HITS)
    off = torch.cumsum(kept, 0) - kept
    n_hits = int(kept.sum().item())
    m = max(n_hits, 1)
    hit_t = torch.empty(m, dtype=torch.float64, device="cuda")
    hit_key = torch.empty(m, dtype=torch.int64, device="cuda")
    hit_scale = torch.empty(m, dtype=torch.float64, device="cuda")
    hit_alpha = torch.empty(m, dtype=torch.float64, device="cuda")
    hit_c = torch.empty((m, 3), dtype=torch.float32, device="cuda")
    dx, dy, _ = model.spec.dims
    if S:
        v = model.dev("seg_voxel").to(torch.int64)
        seg_lin = (v[:, 0] + dx * (v[:, 1] + dy * v[:, 2])).to(torch.int32)
    else:
        seg_lin = torch.zeros(1, dtype=torch.int32, device="cuda")
    img_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
    stats_d = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
    _lib.check(L.lvx_brute_render(C.byref(plan.cam), C.byref(plan.mdl), C.byref(plan.par), C.byref(plan.lod),
                                  C.c_int64(S), _lib.ptr(seg_lin), _lib.ptr(count), _lib.ptr(off), _lib.ptr(hit_t),
                                  _lib.ptr(hit_key), _lib.ptr(hit_scale), _lib.ptr(hit_alpha), _lib.ptr(hit_c),
                                  _lib.ptr(img_d), _lib.ptr(stats_d), st))
    e1.record()
    img = img_d.cpu().numpy()
    tot = stats_d.sum(dim=0).cpu()
    stats = {"rays": W * H, "voxel_steps": 0, "intersection_tests": int(tot[1]), "ms": float(e0.elapsed_time(e1)),
             "workers": 1, "window_overflow": int(tot[2])}
    return Frame(image=img, stats=stats)


def _as_float_image(img) -> np.ndarray:
    if hasattr(img, "image"):
        img = img.image
    arr = np.asarray(img)
    if arr.dtype == np.uint8:
        return arr.astype(np.float64) / 255.0
    return arr.astype(np.float64)


def image_compare(a, b, tol: float = 2.0 / 255.0) -> dict:
    """Channel-wise comparison of two images or Frames (metrics.py:122-143): maximum channel
    difference, fraction of pixels whose every channel is within `tol`, PSNR against a unit peak."""
    ia, ib = _as_float_image(a), _as_float_image(b)
    if ia.shape != ib.shape:
        raise ValueError(f"image shapes differ: {ia.shape} vs {ib.shape}")
    if ia.ndim != 3:
        raise ValueError("expected (height, width, channels) images")
    diff = np.abs(ia - ib)
    if diff.size == 0:
        return {"max_diff": 0.0, "fraction_close": 1.0, "psnr": math.inf}
    mse = float(np.mean(diff * diff))
    return {"max_diff": float(diff.max()), "fraction_close": float(np.mean(np.all(diff <= tol, axis=2))),
            "psnr": math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)}


def memory_report(model) -> dict:
    """Exact byte accounting of the encoded model (metrics.py:149-160)."""
    v, s, w = model.voxel_count, model.segment_count, model.record_width
    return {"header_bytes": 5 * v, "segment_bytes": w * s, "total": 5 * v + w * s, "bytes_per_segment": w}
