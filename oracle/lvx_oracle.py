"""ctypes front end of oracle/liblvx_oracle.so (the C restatement of the
reference's hot path).  TEST INFRASTRUCTURE ONLY: importable from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs.

Function names and argument meaning follow the reference
(/root/reference/pkg/src/linevox): build_voxel_model (voxelizer.py:397-488),
compute_density_level0 / build_octree (lod.py:82-119), render (raycast.py:468-521
-> _kernels.py:735-923), precompute_voxel_ao (illumination.py:193-214).
Inputs and outputs are plain numpy arrays / dicts so the module has no
dependency on the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblvx_oracle.so")
_lib = None

OPACITY_MODES = {"constant": 0, "transfer": 1, "distance-scaled": 2}
SHADOW_MODES = {"none": 0, "hard": 1, "replines": 2, "cone": 3}
AO_MODES = {"none": 0, "hemisphere-geometry": 1, "density-rays": 2, "precomputed": 3}


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no GPU, no reference sources involved)."""
    src = os.path.join(_HERE, "lvx_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", _HERE, "-s", "liblvx_oracle.so"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _lib.lvo_clip_batch.restype = C.c_int64
        _lib.lvo_build_from_chords.restype = C.c_int64
        _lib.lvo_dda_collect.restype = C.c_int64
        _lib.lvo_sample_trilinear.restype = C.c_double
        _lib.lvo_cone_blocking.restype = C.c_double
        _lib.lvo_ao_density_point.restype = C.c_double
        _lib.lvo_shade_scalar.restype = C.c_double
        _lib.lvo_render_rows.restype = C.c_int
        _lib.lvo_record_width.restype = C.c_int
        _lib.lvo_num_threads.restype = C.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def num_threads() -> int:
    return int(lib().lvo_num_threads())


def record_width(n_bins: int) -> int:
    return int(lib().lvo_record_width(C.c_int(int(n_bins))))


def default_transfer_table() -> np.ndarray:
    """voxelizer.py:292-303"""
    t = np.linspace(0.0, 1.0, 256)
    cold = np.array([0.231, 0.299, 0.754])
    mid = np.array([0.865, 0.865, 0.865])
    warm = np.array([0.706, 0.016, 0.150])
    table = np.empty((256, 4), dtype=np.float32)
    lo = t < 0.5
    table[lo, :3] = cold + (t[lo, None] * 2.0) * (mid - cold)
    table[~lo, :3] = mid + ((t[~lo, None] - 0.5) * 2.0) * (warm - mid)
    table[:, 3] = 1.0
    return table


# --- voxelizer ------------------------------------------------------------------

def clip_batch(pts, attrs, curve_off, dims):
    """_clip_batch (voxelizer.py:213-263): (vox, p_in, p_out, a_in, a_out, curve, within)."""
    pts, attrs, curve_off = _f64(pts), _f64(attrs), _i64(curve_off)
    d = _i64(dims)
    n_curves = curve_off.size - 1
    cap = max(16, int(pts.shape[0]) * 2)
    while True:
        vox = np.empty((cap, 3), np.int64)
        p_in = np.empty((cap, 3))
        p_out = np.empty((cap, 3))
        a_in = np.empty(cap)
        a_out = np.empty(cap)
        curve = np.empty(cap, np.int64)
        within = np.empty(cap, np.int64)
        n = lib().lvo_clip_batch(_p(pts), _p(attrs), _p(curve_off), C.c_int64(n_curves), _p(d),
                                 C.c_int64(cap), _p(vox), _p(p_in), _p(p_out), _p(a_in),
                                 _p(a_out), _p(curve), _p(within))
        if n <= cap:
            break
        cap = int(n)
    return (vox[:n], p_in[:n], p_out[:n], a_in[:n], a_out[:n], curve[:n], within[:n])


def build_voxel_model(pts, attrs, curve_off, dims, n_bins=32, transfer_table=None):
    """build_voxel_model (voxelizer.py:397-488) on a concatenated curve batch.

    Returns a namespace with the reference's VoxelModel array fields."""
    dims = tuple(int(x) for x in dims)
    vox, p_in, p_out, a_in, a_out, curve, within = clip_batch(pts, attrs, curve_off, dims)
    n = vox.shape[0]
    V = dims[0] * dims[1] * dims[2]
    w = record_width(n_bins)
    m = max(n, 1)
    counts = np.zeros(V, np.uint8)
    offsets = np.zeros(V, np.uint32)
    packed = np.zeros(m * w, np.uint8)
    dropped = np.zeros(1, np.int64)
    seg_voxel = np.zeros((m, 3), np.int32)
    seg_a = np.zeros((m, 3), np.float32)
    seg_b = np.zeros((m, 3), np.float32)
    seg_attr = np.zeros(m, np.uint8)
    seg_lid = np.zeros(m, np.uint8)
    fi = np.zeros(m, np.uint8)
    bi = np.zeros(m, np.uint16)
    fo = np.zeros(m, np.uint8)
    bo = np.zeros(m, np.uint16)
    seg_curve = np.zeros(m, np.int32)
    seg_order = np.zeros(m, np.int32)
    d = _i64(dims)
    S = lib().lvo_build_from_chords(
        C.c_int64(n), _p(vox), _p(p_in), _p(p_out), _p(a_in), _p(a_out), _p(curve), _p(within),
        _p(d), C.c_int(int(n_bins)), _p(counts), _p(offsets), _p(packed), _p(dropped),
        _p(seg_voxel), _p(seg_a), _p(seg_b), _p(seg_attr), _p(seg_lid), _p(fi), _p(bi), _p(fo),
        _p(bo), _p(seg_curve), _p(seg_order))
    if S < 0:
        raise AssertionError("chord endpoint off every face")
    table = default_transfer_table() if transfer_table is None else np.asarray(
        transfer_table, dtype=np.float32)
    return SimpleNamespace(
        dims=dims, n_bins=int(n_bins), counts=counts, offsets=offsets, packed=packed[:S * w].copy(),
        transfer_table=table, seg_voxel=seg_voxel[:S].copy(), seg_a=seg_a[:S].copy(),
        seg_b=seg_b[:S].copy(), seg_attr=seg_attr[:S].copy(), seg_lid=seg_lid[:S].copy(),
        seg_face_in=fi[:S].copy(), seg_bin_in=bi[:S].copy(), seg_face_out=fo[:S].copy(),
        seg_bin_out=bo[:S].copy(), dropped_overflow=int(dropped[0]),
        seg_curve=seg_curve[:S].copy(), seg_order=seg_order[:S].copy(), ao=None,
        segment_count=int(S))


# --- LoD --------------------------------------------------------------------------

def compute_density_level0(model) -> np.ndarray:
    dx, dy, dz = model.dims
    out = np.zeros(dx * dy * dz, np.float32)
    S = int(model.seg_attr.shape[0])
    if S:
        lib().lvo_density_l0(C.c_int64(S), _p(np.ascontiguousarray(model.seg_a)),
                             _p(np.ascontiguousarray(model.seg_b)), _p(model.seg_attr),
                             _p(np.ascontiguousarray(model.seg_voxel)),
                             _p(np.ascontiguousarray(model.transfer_table, dtype=np.float32)),
                             _p(_i64(model.dims)), _p(out))
    return out.reshape(dz, dy, dx)


def coarsen(field: np.ndarray) -> np.ndarray:
    field = np.ascontiguousarray(field, dtype=np.float32)
    dz, dy, dx = field.shape
    out = np.empty(((dz + 1) // 2, (dy + 1) // 2, (dx + 1) // 2), np.float32)
    lib().lvo_coarsen(_p(field), _p(_i64([dx, dy, dz])), _p(out))
    return out


def build_octree(level0: np.ndarray) -> list:
    levels = [np.ascontiguousarray(level0, dtype=np.float32)]
    while levels[-1].shape != (1, 1, 1):
        levels.append(coarsen(levels[-1]))
    return levels


def octree_args(levels):
    """raycast.py:369-388 (flat f32, offsets i64[L+1], dims i64[L,3] as dx,dy,dz, L)."""
    if levels is None:
        return (np.zeros(1, np.float32), np.zeros(2, np.int64), np.ones((1, 3), np.int64), 1)
    offs, dims, parts = [0], [], []
    for lvl in levels:
        dz, dy, dx = lvl.shape
        dims.append((dx, dy, dz))
        parts.append(np.ascontiguousarray(lvl.reshape(-1)))
        offs.append(offs[-1] + lvl.size)
    return (np.concatenate(parts).astype(np.float32), np.asarray(offs, np.int64),
            np.asarray(dims, np.int64), len(levels))


def occupancy_dilated(model) -> np.ndarray:
    rx, ry, rz = model.dims
    out = np.zeros((rx + 2) * (ry + 2) * (rz + 2), np.uint8)
    lib().lvo_occupancy_dilated(_p(model.counts), _p(_i64(model.dims)), _p(out))
    return out


# --- primitives ---------------------------------------------------------------------

def dda_collect(o, d, dims, pad=0):
    o, d = _f64(o), _f64(d)
    rx, ry, rz = (int(x) for x in dims)
    cap = rx + ry + rz + 6 * (pad + 2)
    vox = np.empty((cap, 3), np.int64)
    t = np.empty((cap, 2))
    n = lib().lvo_dda_collect(*(C.c_double(float(v)) for v in (*o, *d)), C.c_int64(rx),
                              C.c_int64(ry), C.c_int64(rz), C.c_int64(pad), C.c_int64(cap),
                              _p(vox), _p(t))
    return vox[:n], t[:n]


def intersect_tube(o, d, a, b, r, f32_axis=True):
    out = np.zeros(6)
    if f32_axis:
        lib().lvo_intersect_tube_f32(_p(_f64(o)), _p(_f64(d)),
                                     _p(np.ascontiguousarray(a, dtype=np.float32)),
                                     _p(np.ascontiguousarray(b, dtype=np.float32)),
                                     C.c_double(float(r)), _p(out))
    else:
        lib().lvo_intersect_tube_f64(_p(_f64(o)), _p(_f64(d)), _p(_f64(a)), _p(_f64(b)),
                                     C.c_double(float(r)), _p(out))
    return out


def intersect_sphere(o, d, c, r):
    out = np.zeros(6)
    lib().lvo_intersect_sphere(_p(_f64(o)), _p(_f64(d)), _p(_f64(c)), C.c_double(float(r)), _p(out))
    return out


def shade_scalar(n, l, v, ka, kd, ks, shininess):
    return float(lib().lvo_shade_scalar(_p(_f64(n)), _p(_f64(l)), _p(_f64(v)), C.c_double(ka),
                                        C.c_double(kd), C.c_double(ks), C.c_double(shininess)))


def sample_trilinear(flat, off, ldx, ldy, ldz, scale, p):
    flat = np.ascontiguousarray(flat, dtype=np.float32)
    return float(lib().lvo_sample_trilinear(_p(flat), C.c_int64(off), C.c_int64(ldx), C.c_int64(ldy),
                                            C.c_int64(ldz), C.c_double(scale),
                                            *(C.c_double(float(x)) for x in p)))


def cone_blocking(p, l, levels, eps=0.01):
    flat, off, dims, L = octree_args(levels)
    gx, gy, gz = (float(x) for x in dims[0])
    return float(lib().lvo_cone_blocking(*(C.c_double(float(x)) for x in (*p, *l)), _p(flat), _p(off),
                                         _p(dims), C.c_int64(L), C.c_double(gx), C.c_double(gy),
                                         C.c_double(gz), C.c_double(eps)))


def ao_density_point(p, n, levels, n_rays, radius, step, hemisphere=1):
    flat, off, dims, _ = octree_args(levels)
    gx, gy, gz = (float(x) for x in dims[0])
    return float(lib().lvo_ao_density_point(*(C.c_double(float(x)) for x in (*p, *n)),
                                            C.c_int64(n_rays), C.c_double(radius), C.c_double(step),
                                            C.c_int(hemisphere), _p(flat), _p(off), _p(dims),
                                            C.c_double(gx), C.c_double(gy), C.c_double(gz)))


def fibonacci_dir(i, n, hemisphere, jitter=0.0):
    out = np.zeros(3)
    lib().lvo_fibonacci_dir(C.c_int64(i), C.c_int64(n), C.c_int(hemisphere), C.c_double(jitter), _p(out))
    return out


def precompute_voxel_ao(model, levels, n_rays=100, radius=5.0, step=1.0, threads=0) -> np.ndarray:
    rx, ry, rz = model.dims
    flat, off, dims, _ = octree_args(levels)
    out = np.zeros(rx * ry * rz, np.float32)
    lib().lvo_precompute_ao(_p(model.counts), _p(_i64(model.dims)), C.c_int64(n_rays),
                            C.c_double(radius), C.c_double(step), _p(flat), _p(off), _p(dims),
                            _p(out), C.c_int(threads))
    return out.reshape(rz, ry, rx)


# --- frame ---------------------------------------------------------------------------

def camera_args(position, target, up, fov, width, height):
    """Camera.basis + _camera_args (raycast.py:63-76, 335-341)."""
    position, target, up = _f64(position), _f64(target), _f64(up)
    fwd = target - position
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, up)
    right = right / np.linalg.norm(right)
    upv = np.cross(right, fwd)
    tan_half = float(np.tan(np.radians(fov) * 0.5))
    return (np.ascontiguousarray(position), np.ascontiguousarray(right),
            np.ascontiguousarray(upv), np.ascontiguousarray(fwd), tan_half,
            width / height, int(width), int(height))


def default_camera(dims, width=640, height=360):
    """raycast.py:441-448 -> dict(position, target, up, fov, width, height)."""
    center = np.asarray(dims, dtype=np.float64) * 0.5
    dist = 1.9 * float(max(dims))
    position = center + np.array([0.0, -dist, 0.42 * dist])
    return dict(position=position, target=center, up=(0.0, 0.0, 1.0), fov=45.0,
                width=width, height=height)


class RepLevel:
    def __init__(self, valid, a, b, weight):
        self.valid, self.a, self.b, self.weight = valid, a, b, weight


def build_rep_lines(model, n_levels: int, adjacency: bool = True):
    """build_rep_lines (lod.py:224-284): list indexed by level, entry 0 is None."""
    n_bins = int(model.n_bins)
    levels = [None]
    cur_a = np.asarray(model.seg_a, dtype=np.float64)
    cur_b = np.asarray(model.seg_b, dtype=np.float64)
    cur_vox = np.asarray(model.seg_voxel, dtype=np.int64)
    d = cur_b - cur_a
    cur_w = np.sqrt((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
    cur_dims = tuple(int(x) for x in model.dims)
    L = lib()
    for level in range(1, int(n_levels)):
        pd = tuple((x + 1) // 2 for x in cur_dims)
        size = float(1 << level)
        pvox = cur_vox // 2
        plin = pvox[:, 0] + pd[0] * (pvox[:, 1] + pd[1] * pvox[:, 2])
        order = np.argsort(plin, kind="stable")
        n_parent = pd[0] * pd[1] * pd[2]
        valid = np.zeros(n_parent, dtype=np.uint8)
        rep_a = np.zeros((n_parent, 3), dtype=np.float32)
        rep_b = np.zeros((n_parent, 3), dtype=np.float32)
        rep_w = np.zeros(n_parent, dtype=np.float32)
        a_s = np.ascontiguousarray(cur_a[order])
        b_s = np.ascontiguousarray(cur_b[order])
        w_s = np.ascontiguousarray(cur_w[order])
        p_s = np.ascontiguousarray(plin[order])
        pdv = np.asarray(pd, dtype=np.int64)
        L.lvo_rep_level(C.c_int64(a_s.shape[0]), _p(a_s), _p(b_s), _p(w_s), _p(p_s), _p(pdv), C.c_double(size),
                        C.c_int64(n_bins), _p(valid), _p(rep_a), _p(rep_b), _p(rep_w))
        if adjacency:
            L.lvo_rep_adjacency(_p(pdv), C.c_double(size), C.c_int64(n_bins), _p(valid), _p(rep_a), _p(rep_b))
        levels.append(RepLevel(valid.astype(bool), rep_a, rep_b, rep_w))
        keep = np.nonzero(valid)[0]
        cur_a = rep_a[keep].astype(np.float64)
        cur_b = rep_b[keep].astype(np.float64)
        cur_w = rep_w[keep].astype(np.float64)
        cur_vox = np.stack([keep % pd[0], (keep // pd[0]) % pd[1], keep // (pd[0] * pd[1])], axis=1)
        cur_dims = pd
    return levels


def _rep_level_args(levels, dims, level):
    level = max(1, min(int(level), len(levels) - 1))
    lvl = levels[level]
    ld = np.asarray([-(-int(g) // (1 << level)) for g in dims], dtype=np.int64)
    return (np.ascontiguousarray(lvl.valid, dtype=np.uint8), np.ascontiguousarray(lvl.a, dtype=np.float32),
            np.ascontiguousarray(lvl.b, dtype=np.float32), np.ascontiguousarray(lvl.weight, dtype=np.float32), ld,
            float(1 << level))


def replines_shadow(point, light, levels, grid_dims, level=1, tube_radius=0.3, normal=None) -> int:
    """illumination.replines_shadow (illumination.py:115-139): 1 if the point sees the light."""
    if not 1 <= level < len(levels):
        raise ValueError(f"level must be in [1, {len(levels) - 1}], got {level}")
    o = _f64(point)
    if normal is not None:
        nn = _f64(normal)
        o = o + 1e-3 * (nn / np.linalg.norm(nn))
    to_light = _f64(light) - o
    max_t = float(np.linalg.norm(to_light))
    if max_t == 0.0:
        return 1
    d = to_light / max_t
    valid, a, b, w, ld, size = _rep_level_args(levels, grid_dims, level)
    fn = lib().lvo_replines_blocked
    fn.restype = C.c_int
    blocked = fn(_p(o), _p(d), C.c_double(max_t), _p(valid), _p(a), _p(b), _p(w), _p(ld), C.c_double(size),
                 C.c_double(float(tube_radius) * size))
    return 0 if blocked else 1


def hard_shadow(point, light, model, radius=0.3, normal=None, joint_spheres=True) -> int:
    """illumination.hard_shadow (illumination.py:96-112): 1 if the point sees the light position."""
    o = _f64(point)
    if normal is not None:
        nn = _f64(normal)
        o = o + 1e-3 * (nn / np.linalg.norm(nn))
    to_light = _f64(light) - o
    max_t = float(np.linalg.norm(to_light))
    if max_t == 0.0:
        return 1
    d = to_light / max_t
    rx, ry, rz = model.dims
    seg_a = np.ascontiguousarray(model.seg_a, dtype=np.float32)
    seg_b = np.ascontiguousarray(model.seg_b, dtype=np.float32)
    fn = lib().lvo_geometry_blocked
    fn.restype = C.c_int
    blocked = fn(_p(o), _p(d), C.c_double(max_t), C.c_int64(rx), C.c_int64(ry), C.c_int64(rz),
                 _p(model.counts), _p(model.offsets), _p(seg_a), _p(seg_b), C.c_double(float(radius)),
                 C.c_int(1 if joint_spheres else 0))
    return 0 if blocked else 1


def ao_hemisphere_geometry(point, normal, model, n_rays=100, radius=15.0, tube_radius=0.3, jitter=0.0) -> float:
    """illumination.ao_hemisphere_geometry (illumination.py:158-173)."""
    p = _f64(point)
    nn = _f64(normal)
    nn = nn / np.linalg.norm(nn)
    rx, ry, rz = model.dims
    seg_a = np.ascontiguousarray(model.seg_a, dtype=np.float32)
    seg_b = np.ascontiguousarray(model.seg_b, dtype=np.float32)
    fn = lib().lvo_ao_hemisphere_point
    fn.restype = C.c_double
    return float(fn(_p(p), _p(nn), C.c_int64(int(n_rays)), C.c_double(float(radius)), C.c_double(float(jitter)),
                    C.c_int64(rx), C.c_int64(ry), C.c_int64(rz), _p(model.counts), _p(model.offsets),
                    _p(seg_a), _p(seg_b), C.c_double(float(tube_radius))))


def render(camera: dict, model, levels=None, *, tube_radius=0.3, opacity_mode="constant",
           base_opacity=1.0, tau=0.95, neighbor=True, joint_spheres=True, shadow_mode="none",
           ao_mode="none", background=(0.0, 0.0, 0.0, 1.0), light_dir=None, ambient=0.2,
           diffuse=0.7, specular=0.3, shininess=32.0, ao_rays=25, ao_radius=15.0, threads=0,
           rows=None, replines=None, shadow_rep_level=2):
    """render_frame (raycast.py:468-521): returns (image (H,W,4) f32, stats dict).

    `rows=(y0, y1[, step])` renders only rows y0, y0+step, ... < y1 (bounded CPU timing)."""
    cam = camera_args(**camera)
    W, H = cam[6], cam[7]
    rx, ry, rz = model.dims
    flat, off, dims, L = octree_args(levels)
    if light_dir is None:
        headlight, light = 1, np.zeros(3)
    else:
        headlight, light = 0, _f64(light_dir) / np.linalg.norm(_f64(light_dir))
    ao = getattr(model, "ao", None)
    ao_flat = (np.ascontiguousarray(np.asarray(ao).reshape(-1), dtype=np.float32)
               if ao is not None else np.zeros(1, np.float32))
    if AO_MODES[ao_mode] == 3 and ao is None:
        raise ValueError("precomputed AO requested but the model carries none")
    occ = getattr(model, "_occ_cache", None)
    if occ is None:
        occ = occupancy_dilated(model)
        try:
            model._occ_cache = occ
        except AttributeError:
            pass
    img = np.zeros((H, W, 4), np.float32)
    stats = np.zeros((H, 3), np.int64)
    y0, y1, ystep = (0, H, 1) if rows is None else (tuple(rows) + (1,))[:3]
    bg = _f64(background)
    table = np.ascontiguousarray(model.transfer_table, dtype=np.float32)
    seg_a = np.ascontiguousarray(model.seg_a, dtype=np.float32)
    seg_b = np.ascontiguousarray(model.seg_b, dtype=np.float32)
    rep_keep = None
    if SHADOW_MODES[shadow_mode] == 2:
        if replines is None:
            raise ValueError("replines shadows need a representative-line field")
        rep_keep = _rep_level_args(replines, model.dims, shadow_rep_level)
        lib().lvo_set_replines(_p(rep_keep[0]), _p(rep_keep[1]), _p(rep_keep[2]), _p(rep_keep[3]), _p(rep_keep[4]),
                               C.c_double(rep_keep[5]))
    rc = lib().lvo_render_rows(
        _p(cam[0]), _p(cam[1]), _p(cam[2]), _p(cam[3]), C.c_double(cam[4]), C.c_double(cam[5]),
        C.c_int64(W), C.c_int64(H), C.c_int64(y0), C.c_int64(y1), C.c_int64(max(1, ystep)), C.c_int64(rx), C.c_int64(ry),
        C.c_int64(rz), _p(model.counts), _p(model.offsets), _p(seg_a), _p(seg_b),
        _p(model.seg_attr), _p(model.seg_lid), _p(table), _p(occ), C.c_double(tube_radius),
        C.c_int64(OPACITY_MODES[opacity_mode]), C.c_double(base_opacity), C.c_double(tau),
        C.c_int64(1 if neighbor else 0), C.c_int64(1 if joint_spheres else 0),
        C.c_double(ambient), C.c_double(diffuse), C.c_double(specular), C.c_double(shininess),
        C.c_int64(headlight), _p(light), _p(bg), C.c_int64(SHADOW_MODES[shadow_mode]),
        C.c_int64(AO_MODES[ao_mode]), _p(flat), _p(off), _p(dims), C.c_int64(L), _p(ao_flat),
        C.c_int64(int(ao_rays)), C.c_double(float(ao_radius)), _p(img), _p(stats), C.c_int(threads))
    if rc != 0:
        raise NotImplementedError("oracle does not restate shadow_mode='replines'")
    st = {"rays": W * H, "voxel_steps": int(stats[:, 0].sum()),
          "intersection_tests": int(stats[:, 1].sum()),
          "window_overflow": int(stats[:, 2].sum()), "neighbor": bool(neighbor)}
    return img, st
