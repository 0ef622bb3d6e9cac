"""Per-pixel ray casting over the two-level voxel model: the reference's
`render_frame` (raycast.py:468-521) with `render_rows` (_kernels.py:735-923)
replaced by the sm_100a kernel behind `lvx_render`.

Host-side ray setup (camera basis, tan(fov/2), light normalisation) is the same
float64 numpy arithmetic as the reference (raycast.py:63-76, 335-341, 427-433), so
the kernel receives bit-identical camera arguments.

The small reference operations `traverse_voxels`, `intersect_ray_tube` and
`intersect_ray_sphere` run through the device probes so tests exercise the same
device functions the frame kernel is built from.
"""
from __future__ import annotations

import os

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .lod import DensityOctree, build_lod
from .voxelizer import VoxelModel

_OPACITY_MODES = {"constant": 0, "transfer": 1, "distance-scaled": 2}
_SHADOW_MODES = {"none": 0, "hard": 1, "replines": 2, "cone": 3}
_AO_MODES = {"none": 0, "hemisphere-geometry": 1, "density-rays": 2, "precomputed": 3}

TILE_W, TILE_H = 8, 4  # one warp = one 8x4 pixel tile


@dataclass
class Camera:
    """Pinhole camera in grid-local units; fov is vertical, in degrees (raycast.py:40-87)."""

    position: Sequence[float]
    target: Sequence[float]
    up: Sequence[float] = (0.0, 0.0, 1.0)
    fov: float = 45.0
    width: int = 640
    height: int = 360

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.target = np.asarray(self.target, dtype=np.float64)
        self.up = np.asarray(self.up, dtype=np.float64)
        if self.position.shape != (3,) or self.target.shape != (3,) or self.up.shape != (3,):
            raise ValueError("camera vectors must have 3 components")
        if not 0.0 < self.fov < 180.0:
            raise ValueError("fov must be in (0, 180) degrees")
        if self.width < 1 or self.height < 1:
            raise ValueError("image dims must be >= 1")
        self.basis()

    def basis(self):
        """Right/up/forward unit vectors of the view frame."""
        fwd = self.target - self.position
        fn = np.linalg.norm(fwd)
        if fn < 1e-12:
            raise ValueError("camera position and target coincide")
        fwd = fwd / fn
        right = np.cross(fwd, self.up)
        rn = np.linalg.norm(right)
        if rn < 1e-9:
            raise ValueError("up vector is parallel to the view direction")
        right = right / rn
        up = np.cross(right, fwd)
        return right, up, fwd

    def ray(self, x: int, y: int):
        """Primary ray through the centre of pixel (x, y); y runs downward."""
        right, up, fwd = self.basis()
        tan_half = np.tan(np.radians(self.fov) * 0.5)
        aspect = self.width / self.height
        ndc_x = ((x + 0.5) / self.width * 2.0 - 1.0) * tan_half * aspect
        ndc_y = (1.0 - (y + 0.5) / self.height * 2.0) * tan_half
        d = fwd + ndc_x * right + ndc_y * up
        d = d / np.linalg.norm(d)
        return self.position.copy(), d


@dataclass
class RenderParams:
    """raycast.py:90-129 (same fields, defaults and validation)."""

    tube_radius: float = 0.3
    opacity_mode: str = "constant"
    base_opacity: float = 1.0
    tau: float = 0.95
    neighbor_mode: str = "auto"
    shadow_mode: str = "none"
    ao_mode: str = "none"
    background: Sequence[float] = (0.0, 0.0, 0.0, 1.0)
    joint_spheres: bool = True
    light_dir: Optional[Sequence[float]] = None  # headlight unless a direction is given
    ambient: float = 0.2
    diffuse: float = 0.7
    specular: float = 0.3
    shininess: float = 32.0
    ao_rays: int = 25
    ao_radius: float = 15.0
    shadow_rep_level: int = 2

    def __post_init__(self):
        if not 0.0 < self.tube_radius <= 0.5:
            raise ValueError("tube_radius must be in (0, 0.5] voxel units")
        if self.opacity_mode not in _OPACITY_MODES:
            raise ValueError("opacity_mode must be one of %s" % sorted(_OPACITY_MODES))
        if not 0.0 < self.base_opacity <= 1.0:
            raise ValueError("base_opacity must be in (0, 1]")
        if not 0.0 < self.tau <= 1.0:
            raise ValueError("tau must be in (0, 1]")
        if self.neighbor_mode not in ("off", "on", "auto"):
            raise ValueError("neighbor_mode must be off, on or auto")
        if self.shadow_mode not in _SHADOW_MODES:
            raise ValueError("shadow_mode must be one of %s" % sorted(_SHADOW_MODES))
        if self.ao_mode not in _AO_MODES:
            raise ValueError("ao_mode must be one of %s" % sorted(_AO_MODES))
        bg = np.asarray(self.background, dtype=np.float64)
        if bg.shape != (4,):
            raise ValueError("background must be RGBA")
        self.background = bg


@dataclass
class HitRecord:
    t_in: float
    t_out: float
    normal: np.ndarray
    voxel: Optional[tuple] = None
    local_line_id: int = 0
    attr_index: int = 0
    kind: str = "tube"


@dataclass
class Frame:
    image: np.ndarray  # (H, W, 4) float32, premultiplied RGBA in [0,1]
    stats: dict = field(default_factory=dict)

    @property
    def width(self) -> int:
        return self.image.shape[1]

    @property
    def height(self) -> int:
        return self.image.shape[0]

    def to_rgba8(self) -> np.ndarray:
        return np.clip(np.rint(self.image * 255.0), 0, 255).astype(np.uint8)


# --- point probes -----------------------------------------------------------------

def _as_ray(ray):
    origin, direction = ray
    o = np.asarray(origin, dtype=np.float64)
    d = np.asarray(direction, dtype=np.float64)
    n = np.linalg.norm(d)
    if n == 0.0:
        raise ValueError("ray direction must be non-zero")
    return o, d / n


def traverse_voxels(ray, spec, pad: int = 0):
    """Ordered (voxel, t_enter, t_exit) triples of the DDA walk (raycast.py:170-181)."""
    o, d = _as_ray(ray)
    return probe_dda(o, d, tuple(int(v) for v in getattr(spec, "dims", spec)), pad)


def probe_dda(o, d, dims, pad: int = 0):
    """dda_collect (_kernels.py:164-256) for one ray with a unit direction `d` taken as is."""
    torch = _lib.require_device()
    cap = dims[0] + dims[1] + dims[2] + 6 * (pad + 2)
    vox = torch.empty((cap, 3), dtype=torch.int64, device="cuda")
    t = torch.empty((cap, 2), dtype=torch.float64, device="cuda")
    n = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().lvx_probe_dda(_lib.f64x3(o), _lib.f64x3(d), _lib.i32x3(dims),
                                        C.c_int32(int(pad)), C.c_int64(cap), _lib.ptr(vox),
                                        _lib.ptr(t), _lib.ptr(n), _lib.stream_ptr()))
    k = int(n.item())
    vox, t = vox[:k].cpu().numpy(), t[:k].cpu().numpy()
    return [(tuple(int(v) for v in vox[i]), float(t[i, 0]), float(t[i, 1])) for i in range(k)]


def probe_tubes(rays: np.ndarray, a: np.ndarray, b: np.ndarray, radius: float,
                f32_axis: bool = False) -> np.ndarray:
    """Batched tube test: rays (n,6) = origin|unit direction, endpoints (n,3).
    Returns (n,6) = hit, t_in, t_out, normal.  f32_axis selects the frame-kernel
    specialisation (float32 endpoints, float32 axis arithmetic)."""
    torch = _lib.require_device()
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    n = rays.shape[0]
    dt = np.float32 if f32_axis else np.float64
    a_d, b_d = _lib.to_device(np.asarray(a).reshape(-1, 3), dt), _lib.to_device(np.asarray(b).reshape(-1, 3), dt)
    out = torch.empty((max(n, 1), 6), dtype=torch.float64, device="cuda")
    rays_d = _lib.to_device(rays)  # named: a temporary would be recycled by the caching allocator
    _lib.check(_lib.lib().lvx_probe_tube(_lib.ptr(rays_d), _lib.ptr(a_d), _lib.ptr(b_d),
                                         C.c_double(float(radius)), C.c_int32(1 if f32_axis else 0),
                                         C.c_int64(n), _lib.ptr(out), _lib.stream_ptr()))
    return out[:n].cpu().numpy()


def probe_spheres(rays: np.ndarray, centers: np.ndarray, radius: float) -> np.ndarray:
    torch = _lib.require_device()
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    n = rays.shape[0]
    out = torch.empty((max(n, 1), 6), dtype=torch.float64, device="cuda")
    rays_d = _lib.to_device(rays)
    c_d = _lib.to_device(np.asarray(centers).reshape(-1, 3), np.float64)
    _lib.check(_lib.lib().lvx_probe_sphere(
        _lib.ptr(rays_d), _lib.ptr(c_d),
        C.c_double(float(radius)), C.c_int64(n), _lib.ptr(out), _lib.stream_ptr()))
    return out[:n].cpu().numpy()


def intersect_ray_sphere(ray, center, radius: float) -> Optional[HitRecord]:
    o, d = _as_ray(ray)
    if radius <= 0.0:
        raise ValueError("radius must be positive")
    r = probe_spheres(np.concatenate([o, d])[None], np.asarray(center, dtype=np.float64)[None], radius)[0]
    if r[0] == 0.0:
        return None
    return HitRecord(t_in=float(r[1]), t_out=float(r[2]), normal=r[3:6].copy(), kind="joint-sphere")


def intersect_ray_tube(ray, a, b, radius: float) -> Optional[HitRecord]:
    """Slab-clipped cylinder test; degenerate segments fall back to the endpoint
    sphere (raycast.py:184-200).  All-float64 specialisation, like the reference op."""
    o, d = _as_ray(ray)
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if radius <= 0.0:
        raise ValueError("radius must be positive")
    if np.linalg.norm(b - a) < 1e-12:
        return intersect_ray_sphere(ray, a, radius)
    r = probe_tubes(np.concatenate([o, d])[None], a[None], b[None], radius, f32_axis=False)[0]
    if r[0] == 0.0:
        return None
    return HitRecord(t_in=float(r[1]), t_out=float(r[2]), normal=r[3:6].copy(), kind="tube")


def probe_shade(nlv: np.ndarray, ambient, diffuse, specular, shininess) -> np.ndarray:
    """shade_scalar (_kernels.py:316-329) for rows of (normal, light, view) on the device."""
    torch = _lib.require_device()
    nlv = np.ascontiguousarray(nlv, dtype=np.float64).reshape(-1, 9)
    n = nlv.shape[0]
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    nlv_d = _lib.to_device(nlv)
    _lib.check(_lib.lib().lvx_probe_shade(_lib.ptr(nlv_d), C.c_double(float(ambient)), C.c_double(float(diffuse)),
                                          C.c_double(float(specular)), C.c_double(float(shininess)),
                                          C.c_int64(n), _lib.ptr(out), _lib.stream_ptr()))
    return out[:n].cpu().numpy()


def _hit_sort_key(model_dims, hit: HitRecord):
    rx, ry, _ = model_dims
    vx, vy, vz = hit.voxel
    return (hit.t_in, vx + rx * (vy + ry * vz), hit.local_line_id, 0 if hit.kind == "tube" else 1)


def gather_voxel_hits(ray, voxel, model: VoxelModel, params: RenderParams, seen: Optional[dict] = None,
                      t_window=None):
    """Hits owned by `voxel`, in compositing order (raycast.py:224-283): the voxel's own segments
    -- in neighbour mode those of its 26 neighbours too -- are tested (all-float64 tube / sphere
    tests, batched through the device probes) and a hit is kept when its entry parameter lies
    in the voxel's traversal window.  `seen` maps voxel linear index -> bitmask of line ids that
    are already composited; those segments are skipped."""
    o, d = _as_ray(ray)
    voxel = tuple(int(v) for v in voxel)
    dims = model.spec.dims
    if t_window is None:
        pad = 1 if params.neighbor_mode != "off" else 0
        for vox, t0, t1 in traverse_voxels((o, d), model.spec, pad=pad):
            if vox == voxel:
                t_window = (t0, t1)
                break
        if t_window is None:
            return []
    t0, t1 = t_window
    rx, ry, rz = dims
    span = 1 if params.neighbor_mode != "off" else 0
    cand = []  # (segment index, home voxel, lid, attr) in gather order
    for nz in range(voxel[2] - span, voxel[2] + span + 1):
        for ny in range(voxel[1] - span, voxel[1] + span + 1):
            for nx in range(voxel[0] - span, voxel[0] + span + 1):
                if not (0 <= nx < rx and 0 <= ny < ry and 0 <= nz < rz):
                    continue
                lin = nx + rx * (ny + ry * nz)
                base = int(model.offsets[lin])
                for sgi in range(base, base + int(model.counts[lin])):
                    lid = int(model.seg_lid[sgi])
                    if seen is not None and (seen.get(lin, 0) >> lid) & 1:
                        continue
                    cand.append((sgi, (nx, ny, nz), lid, int(model.seg_attr[sgi])))
    if not cand:
        return []
    idx = np.array([c[0] for c in cand])
    a = model.seg_a[idx].astype(np.float64)
    b = model.seg_b[idx].astype(np.float64)
    rays = np.broadcast_to(np.concatenate([o, d]), (len(cand), 6))
    r = float(params.tube_radius)
    degenerate = np.linalg.norm(b - a, axis=1) < 1e-12
    tube = probe_tubes(rays, a, b, r, f32_axis=False)
    sph_a = probe_spheres(rays, a, r)
    sph_b = probe_spheres(rays, b, r) if params.joint_spheres else None
    hits = []
    for k, (_, home, lid, attr) in enumerate(cand):
        # a zero-length chord is tested as the sphere about its start point (raycast.py:193-194)
        rows = [(sph_a[k], "joint-sphere") if degenerate[k] else (tube[k], "tube")]
        if params.joint_spheres:
            rows += [(sph_a[k], "joint-sphere"), (sph_b[k], "joint-sphere")]
        for row, kind in rows:
            if row[0] == 0.0 or not t0 <= row[1] < t1:
                continue
            hits.append(HitRecord(t_in=float(row[1]), t_out=float(row[2]), normal=row[3:6].copy(), voxel=home,
                                  local_line_id=lid, attr_index=attr, kind=kind))
    hits.sort(key=lambda h: _hit_sort_key(dims, h))
    return hits


def shade_local(hit, light, view, ambient=0.2, diffuse=0.7, specular=0.3, shininess=32.0) -> float:
    """Local shading scale (raycast.py:286-294); `hit` may be a HitRecord or a bare normal."""
    n = np.asarray(getattr(hit, "normal", hit), dtype=np.float64)
    row = np.concatenate([n, np.asarray(light, dtype=np.float64), np.asarray(view, dtype=np.float64)])
    return float(probe_shade(row[None], ambient, diffuse, specular, shininess)[0])


def composite(hits, params: RenderParams, transfer_table, ray_dir=(0.0, 0.0, 1.0)) -> np.ndarray:
    """Front-to-back blend of pre-sorted hits; returns premultiplied RGBA (raycast.py:297-332).
    Stops once the accumulated alpha reaches tau, then blends the background underneath."""
    table = np.asarray(transfer_table, dtype=np.float32)
    d = np.asarray(ray_dir, dtype=np.float64)
    d = d / np.linalg.norm(d)
    view = -d
    if params.light_dir is None:
        light = view
    else:
        light = np.asarray(params.light_dir, dtype=np.float64)
        light = light / np.linalg.norm(light)
    hits = list(hits)
    scales = np.zeros(0)
    if hits:
        nlv = np.stack([np.concatenate([np.asarray(h.normal, dtype=np.float64), light, view]) for h in hits])
        scales = probe_shade(nlv, params.ambient, params.diffuse, params.specular, params.shininess)
    mode = _OPACITY_MODES[params.opacity_mode]
    acc = np.zeros(4, dtype=np.float64)
    for h, scale in zip(hits, scales):
        if mode == 0:
            alpha = params.base_opacity
        elif mode == 1:
            alpha = float(table[h.attr_index, 3])
        else:
            alpha = 1.0 - (1.0 - params.base_opacity) ** max(0.0, h.t_out - h.t_in)
        w = (1.0 - acc[3]) * alpha
        acc[:3] += w * float(scale) * table[h.attr_index, :3].astype(np.float64)
        acc[3] += w
        if acc[3] >= params.tau:
            break
    bg = params.background
    acc[:3] += (1.0 - acc[3]) * bg[3] * bg[:3]
    acc[3] += (1.0 - acc[3]) * bg[3]
    return acc


# --- frame ---------------------------------------------------------------------------

def default_camera(dims, width: int = 640, height: int = 360) -> Camera:
    """Camera that frames the whole grid from -y, slightly elevated (raycast.py:441-448)."""
    center = np.asarray(dims, dtype=np.float64) * 0.5
    dist = 1.9 * float(max(dims))
    position = center + np.array([0.0, -dist, 0.42 * dist])
    return Camera(position=position, target=center, up=(0.0, 0.0, 1.0), fov=45.0, width=width,
                  height=height)


def ensure_lod(model: VoxelModel, octree: Optional[DensityOctree], replines, params: RenderParams):
    """Build the octree the requested shadow/AO modes need (raycast.py:451-465)."""
    need_octree = (params.shadow_mode == "cone" or params.ao_mode == "density-rays"
                   or (params.shadow_mode == "replines" and replines is None))
    if need_octree and octree is None:
        octree = build_lod(model)
    if params.shadow_mode == "replines" and replines is None:
        from .lod import build_rep_lines
        replines = build_rep_lines(model, octree)
    if params.ao_mode == "precomputed" and model.ao is None:
        raise ValueError("the model carries no baked AO field; run `linevox precompute-ao` first")
    return octree, replines


def _octree_args(octree: DensityOctree):
    """The flat host layout the reference marshals for its kernels (raycast.py:369-388):
    (flat f32, offsets i64[L+1], dims i64[L,3] as dx,dy,dz, L)."""
    flat = np.concatenate([np.ascontiguousarray(l, dtype=np.float32).reshape(-1) for l in octree.levels])
    off = np.zeros(octree.n_levels + 1, dtype=np.int64)
    off[1:] = np.cumsum([l.size for l in octree.levels])
    dims = np.asarray([octree.dims(l) for l in range(octree.n_levels)], dtype=np.int64)
    return flat, off, dims, octree.n_levels


_BASIS_MEMO = {}  # (position, target, up) bytes -> view frame: a sequence of frames re-uses few cameras


def camera_struct(camera: Camera) -> "_lib.Camera":
    """_camera_args (raycast.py:335-341) as the C struct."""
    key = tuple(np.asarray(v, dtype=np.float64).tobytes() for v in (camera.position, camera.target, camera.up))
    frame = _BASIS_MEMO.get(key)
    if frame is None:
        if len(_BASIS_MEMO) >= 256:
            _BASIS_MEMO.clear()
        frame = _BASIS_MEMO[key] = camera.basis()  # (the numpy cross / norm calls are 0.1 ms per frame)
    right, up, fwd = frame
    s = _lib.Camera()
    for i in range(3):
        s.o[i] = float(camera.position[i])
        s.r[i] = float(right[i])
        s.u[i] = float(up[i])
        s.f[i] = float(fwd[i])
    s.tan_half = float(np.tan(np.radians(camera.fov) * 0.5))
    s.aspect = camera.width / camera.height
    s.width, s.height = int(camera.width), int(camera.height)
    return s


def resolve_neighbor(params: RenderParams, moving: bool) -> int:
    if params.neighbor_mode == "auto":
        return 0 if moving else 1
    return 1 if params.neighbor_mode == "on" else 0


def params_struct(params: RenderParams, neighbor: int) -> "_lib.Params":
    """Mode codes + shading scalars of _illum_args / render_frame (raycast.py:405-438, 498-509)."""
    p = _lib.Params()
    p.tube_r = float(params.tube_radius)
    p.base_alpha = float(params.base_opacity)
    p.tau = float(params.tau)
    p.ka, p.kd, p.ks = float(params.ambient), float(params.diffuse), float(params.specular)
    p.shininess = float(params.shininess)
    if params.light_dir is None:
        p.headlight = 1
        light = np.zeros(3, dtype=np.float64)
    else:
        p.headlight = 0
        light = np.asarray(params.light_dir, dtype=np.float64)
        light = light / np.linalg.norm(light)
    bg = np.asarray(params.background, dtype=np.float64)
    for i in range(3):
        p.light[i] = float(light[i])
    for i in range(4):
        p.bg[i] = float(bg[i])
    p.opacity_mode = _OPACITY_MODES[params.opacity_mode]
    p.neighbor = int(neighbor)
    p.joints = 1 if params.joint_spheres else 0
    p.shadow_mode = _SHADOW_MODES[params.shadow_mode]
    p.ao_mode = _AO_MODES[params.ao_mode]
    p.ao_n_rays = int(params.ao_rays)
    p.ao_radius = float(params.ao_radius)
    return p


def check_modes(params: RenderParams, model: VoxelModel, octree, replines=None):
    """The error behaviour of _illum_args (raycast.py:414-421), plus the modes this
    build does not accelerate."""
    if params.shadow_mode == "replines" and replines is None:
        raise ValueError("replines shadows need a representative-line field")  # raycast.py:416-417
    if params.shadow_mode == "cone" and octree is None:
        raise ValueError("cone shadows need a density octree")
    if params.ao_mode == "density-rays" and octree is None:
        raise ValueError("density-rays AO needs a density octree")
    if params.ao_mode == "precomputed" and getattr(model, "ao", None) is None:
        raise ValueError("precomputed AO requested but the model carries none")


def default_records() -> str:
    """What the wavefront engine reads segments from: LVX_RECORDS=auto|packed|rec.

    "rec": the 32-byte render records (float32 endpoints, built by the voxelizer or decoded from
    the encoded records).  "packed": the encoded records themselves (5 bytes per segment at N = 32,
    decoded in the kernels -- SURVEY.md 8f row 1); the frame is byte-identical.  "auto": packed for a
    model that carries only the encoded arrays (a .vxl file renders without any expansion), rec
    otherwise.  Frames with geometry secondary rays and the tile engine always use "rec"."""
    return os.environ.get("LVX_RECORDS", "auto")


def default_engine() -> str:
    """Frame engine used when none is named: LVX_ENGINE=auto|tile|wavefront.

    Both engines produce the same bytes.  "auto" is the wavefront engine (streaming kernels over
    device queues): C3 1080p neighbour mode 7.8 ms vs 18.8 ms, own-voxel mode 7.3 ms vs 10.9 ms for
    the tile engine (one monolithic kernel) -- except in own-voxel mode on a dense model (more than
    two segments per voxel), where the tile engine is faster.  The tile engine is also the independent
    second implementation the parity tests compare against and the host of the footprint pass."""
    import os
    return os.environ.get("LVX_ENGINE", "auto")


_WF_SCRATCH = {}


_WF_SCALE = {}  # frame shape -> queue scale that shape needed so far


def _wf_scratch(cam, til, scale: float):
    """Scratch buffer of the wavefront engine, cached per device and grown on demand."""
    torch = _lib.require_device()
    need = int(_lib.lib().lvx_render_wf_scratch_bytes(C.byref(cam), C.byref(til), C.c_double(scale)))
    dev = torch.cuda.current_device()
    buf = _WF_SCRATCH.get(dev)
    if buf is None or buf.numel() < need:
        _WF_SCRATCH.pop(dev, None)
        buf = None
        torch.cuda.empty_cache()
        buf = torch.empty(need, dtype=torch.uint8, device="cuda")
        _WF_SCRATCH[dev] = buf
    return buf


class FramePlan:
    """Everything `lvx_render` needs for one (camera, model, params) triple, resolved
    once: C structs plus the device tensors they point into (kept alive here)."""

    def __init__(self, camera: Camera, model: VoxelModel, octree: Optional[DensityOctree],
                 params: RenderParams, neighbor: int, tile_first: int = 0, tile_step: int = 1,
                 compact: bool = False, tile_w: int = TILE_W, tile_h: int = TILE_H,
                 engine: Optional[str] = None, replines=None, records: Optional[str] = None):
        from .illumination import fibonacci_dirs_device
        check_modes(params, model, octree, replines)
        self.engine = engine or default_engine()
        if self.engine == "auto":
            # own-voxel mode on a dense model (several segments per voxel) is the one case the monolithic
            # kernel wins: 1 M lines / 256^3 (5.8 segments per voxel) 7.4 ms vs 10.2 ms; C3 (0.58): 10.9 vs 7.3 ms
            dense = model.segment_count > 2 * model.voxel_count
            self.engine = "tile" if (not neighbor and dense) else "wavefront"
        if self.engine not in ("wavefront", "tile"):
            raise ValueError(f"unknown frame engine {self.engine!r}")
        # queue scale that this frame shape last needed (a frame whose queues overflow is
        # repeated with doubled queues: remember it, render_frame builds a plan per call)
        self._shape = (int(camera.width), int(camera.height), int(tile_first), int(tile_step), bool(compact),
                       int(tile_w), int(tile_h))
        self._scale = _WF_SCALE.get(self._shape, 1.0)
        self.cam = camera_struct(camera)
        self.par = params_struct(params, neighbor)
        geometry_rays = params.shadow_mode == "hard" or params.ao_mode == "hemisphere-geometry"
        self._rep = None
        records = records or default_records()
        if records not in ("auto", "packed", "rec"):
            raise ValueError(f"unknown record source {records!r}")
        can_pack = self.engine == "wavefront" and not geometry_rays and params.shadow_mode != "replines" \
            and model._has("packed")
        self.records = "packed" if can_pack and (records == "packed" or
                                                 (records == "auto" and not model.has_render_caches())) else "rec"
        counts_d, offsets_d, rec_d, table_d, occ_d = model.device_view(
            need_occ=bool(neighbor) or geometry_rays, need_rec=self.records == "rec")
        packed_d = model.dev("packed") if self.records == "packed" else None
        m = _lib.Model()
        m.rx, m.ry, m.rz = model.spec.dims
        m.n_bins = int(model.spec.bins_per_axis)
        m.counts_d, m.offsets_d = counts_d.data_ptr(), offsets_d.data_ptr()
        m.seg_rec_d = rec_d.data_ptr() if rec_d is not None else None
        m.packed_d = packed_d.data_ptr() if packed_d is not None else None
        m.table_d = table_d.data_ptr()
        m.nsum_d = occ_d[0].data_ptr() if occ_d is not None else None
        m.nmask_d = occ_d[1].data_ptr() if occ_d is not None else None
        m.ncell_d = occ_d[2].data_ptr() if occ_d is not None else None
        self.mdl = m
        ao_d = model.ao_device() if params.ao_mode == "precomputed" else None
        dirs_d = fibonacci_dirs_device(params.ao_rays, 1) \
            if params.ao_mode in ("density-rays", "hemisphere-geometry") else None
        if octree is not None:
            self.lod = octree.lod_struct(ao_d, dirs_d)
        else:
            self.lod = _lib.Lod()
            self.lod.n_levels = 0
            self.lod.ao_flat_d = ao_d.data_ptr() if ao_d is not None else None
            self.lod.ao_dirs_d = dirs_d.data_ptr() if dirs_d is not None else None
        if params.shadow_mode == "replines":
            # the level is clamped like _rep_args does (raycast.py:391-402)
            self._rep = replines.level_struct(params.shadow_rep_level, model.spec.dims)
            self.lod.rep = self._rep
        t = _lib.Tiling()
        t.tile_w, t.tile_h = tile_w, tile_h
        t.tile_first, t.tile_step, t.compact = int(tile_first), int(tile_step), 1 if compact else 0
        self.til = t
        self._keep = (counts_d, offsets_d, rec_d, packed_d, table_d, occ_d, ao_d, dirs_d, octree, model)
        self.width, self.height = int(camera.width), int(camera.height)

    def n_my_tiles(self) -> int:
        tx = -(-self.width // self.til.tile_w)
        ty = -(-self.height // self.til.tile_h)
        total = tx * ty
        if self.til.tile_first >= total:
            return 0
        return (total - self.til.tile_first + self.til.tile_step - 1) // self.til.tile_step

    def launch(self, img_d, row_stats_d):
        """Render the frame on the current stream (row_stats_d must be zeroed).

        engine "tile": one monolithic kernel (lvx_render), asynchronous.
        engine "wavefront": streaming kernels over device queues (lvx_render_wf); the call
        returns when the frame is complete.  A queue overflow (LVX_E_RANGE) is retried with
        a larger scratch buffer."""
        L = _lib.lib()
        if self.engine == "tile":
            _lib.check(L.lvx_render(C.byref(self.cam), C.byref(self.mdl), C.byref(self.par),
                                    C.byref(self.lod), C.byref(self.til), _lib.ptr(img_d),
                                    _lib.ptr(row_stats_d), None, _lib.stream_ptr()))
            return
        while True:
            scratch = _wf_scratch(self.cam, self.til, self._scale)
            rc = L.lvx_render_wf(C.byref(self.cam), C.byref(self.mdl), C.byref(self.par),
                                 C.byref(self.lod), C.byref(self.til), _lib.ptr(img_d),
                                 _lib.ptr(row_stats_d), _lib.ptr(scratch), C.c_size_t(scratch.numel()),
                                 C.c_double(self._scale), _lib.stream_ptr())
            if rc == 4 and self._scale < 64.0:  # LVX_E_RANGE: queues too small for this scene
                self._scale *= 2.0
                if self._scale > _WF_SCALE.get(self._shape, 1.0):
                    _WF_SCALE[self._shape] = self._scale
                row_stats_d.zero_()
                continue
            _lib.check(rc)
            return


    def launch_footprint(self, img_d, row_stats_d, voxel_bits_d):
        """Instrumented frame (bench.py): also marks every voxel whose header is read."""
        if self.records != "rec":
            raise ValueError("the footprint pass walks the render records: build the plan with records='rec'")
        _lib.check(_lib.lib().lvx_render_footprint(
            C.byref(self.cam), C.byref(self.mdl), C.byref(self.par), C.byref(self.lod),
            C.byref(self.til), _lib.ptr(img_d), _lib.ptr(row_stats_d), _lib.ptr(voxel_bits_d),
            _lib.stream_ptr()))


def frame_output() -> str:
    """Where `render_frame` lets the kernels write the image: "device" (HBM, then one copy to
    pinned host memory) or "host" (pinned host memory directly, the default: C3 1080p end to end
    10.6 -> 10.2 ms, 4K 35.8 -> 34.2 ms).  LVX_FRAME_OUT overrides."""
    return os.environ.get("LVX_FRAME_OUT", "host")


def render_frame(camera: Camera, model: VoxelModel, octree: Optional[DensityOctree] = None,
                 replines=None, params: Optional[RenderParams] = None, workers: int = 1,
                 moving: bool = False) -> Frame:
    """Render one frame (raycast.py:468-521).  neighbor_mode=auto resolves to off
    while `moving` and on otherwise.  `workers` is accepted for signature
    compatibility; `stats["workers"]` reports the number of GPUs used (1)."""
    if params is None:
        params = RenderParams()
    torch = _lib.require_device()
    neighbor = resolve_neighbor(params, moving)
    plan = FramePlan(camera, model, octree, params, neighbor, replines=replines)
    H, W = camera.height, camera.width
    stats_d = torch.zeros((H, 3), dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    img = torch.empty((H, W, 4), dtype=torch.float32, pin_memory=True)
    if frame_output() == "host":
        # the kernels write each finished pixel (once, 16 bytes) straight into the pinned host
        # image through its device mapping: the transfer rides along with the frame instead
        # of following it
        e0.record()
        plan.launch(img, stats_d)
        e1.record()
    else:
        img_d = torch.empty((H, W, 4), dtype=torch.float32, device="cuda")
        e0.record()
        plan.launch(img_d, stats_d)
        e1.record()
        img.copy_(img_d, non_blocking=True)
    tot = stats_d.sum(dim=0).cpu()  # synchronises
    torch.cuda.current_stream().synchronize()
    stats = {
        "rays": W * H,
        "voxel_steps": int(tot[0]),
        "intersection_tests": int(tot[1]),
        "ms": float(e0.elapsed_time(e1)),
        "workers": 1,
        "window_overflow": int(tot[2]),
        "neighbor": bool(neighbor),
    }
    return Frame(image=img.numpy(), stats=stats)
