"""Density-grid secondary rays: cone soft shadows, density-ray ambient occlusion,
the per-voxel AO bake and its trilinear lookup (illumination.py:142-225 and
_kernels.py:346-445, 541-620 of the reference), evaluated on the GPU.

    lvx_ao_bake           <- precompute_voxel_ao / precompute_ao_kernel
    lvx_probe_cone        <- cone_soft_shadow
    lvx_probe_ao_density  <- ao_density_rays
    lvx_probe_trilinear   <- sample_ao / DensityOctree.sample

    lvx_probe_blocked        <- hard_shadow / geometry_ray_blocked
    lvx_probe_ao_hemisphere  <- ao_hemisphere_geometry / ao_hemisphere_point

    lvx_probe_replines       <- replines_shadow / replines_ray_blocked
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .lod import DensityOctree
from .voxelizer import VoxelModel

_AO_MODES = ("hemisphere-geometry", "density-rays", "precomputed")

__all__ = ["AOField", "AOParams", "ao_density_rays", "ao_hemisphere_geometry", "cone_soft_shadow",
           "hard_shadow", "precompute_voxel_ao", "replines_shadow", "sample_ao"]


@dataclass
class AOParams:
    """Sampling budget for ambient occlusion: `radius` of influence in voxel units,
    march `step` for the density integration (illumination.py:35-57)."""

    n_rays: int = 100
    radius: float = 15.0
    step: float = 1.0
    mode: str = "hemisphere-geometry"

    def __post_init__(self):
        if self.n_rays < 1:
            raise ValueError(f"n_rays must be at least 1, got {self.n_rays}")
        if not self.radius > 0:
            raise ValueError(f"radius must be positive, got {self.radius}")
        if not self.step > 0:
            raise ValueError(f"step must be positive, got {self.step}")
        if self.mode not in _AO_MODES:
            raise ValueError(f"unknown AO mode {self.mode!r}; pick one of {sorted(_AO_MODES)}")


class AOField:
    """Dense per-voxel occlusion in [0,1], shaped (rz, ry, rx) (illumination.py:60-78).
    A field baked on the GPU stays there; `values` downloads it on first access."""

    def __init__(self, values=None, *, _dev=None, _shape=None):
        self._dev = _dev
        self._values = None
        if values is not None:
            v = np.asarray(values, dtype=np.float32)
            if v.ndim != 3:
                raise ValueError(f"expected a 3D field, got shape {v.shape}")
            self._values = v
            self._shape = v.shape
        elif _dev is not None:
            self._shape = tuple(int(s) for s in _shape)
        else:
            raise ValueError("expected a 3D field")

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._dev.cpu().numpy().reshape(self._shape)
        return self._values

    @property
    def shape(self):
        return self._shape

    def flat_device(self):
        if self._dev is None:
            self._dev = _lib.to_device(np.ascontiguousarray(self._values.reshape(-1)))
        return self._dev


def _unit(v, what: str) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    n = float(np.linalg.norm(v))
    if n == 0.0:
        raise ValueError(f"{what} must be a nonzero vector")
    return v / n


_DIRS_CACHE = {}


def fibonacci_dirs_device(n_rays: int, hemisphere: int):
    """Direction lattice of fibonacci_dir (_kernels.py:541-552), built once on the
    host with libm cos/sin (bit-identical to the reference) and kept on the GPU."""
    key = (int(n_rays), int(hemisphere))
    d = _DIRS_CACHE.get(key)
    if d is None:
        d = _lib.to_device(_lib.fibonacci_dirs(n_rays, hemisphere))
        _DIRS_CACHE[key] = d
    return d


def _probe_trilinear(flat_d, off: int, ldims, scale: float, pts: np.ndarray) -> np.ndarray:
    torch = _lib.require_device()
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    n = pts.shape[0]
    pts_d = _lib.to_device(pts)
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    ld = (C.c_int64 * 3)(int(ldims[0]), int(ldims[1]), int(ldims[2]))
    _lib.check(_lib.lib().lvx_probe_trilinear(_lib.ptr(flat_d), C.c_int64(off), ld, C.c_double(scale),
                                              _lib.ptr(pts_d), C.c_int64(n), _lib.ptr(out),
                                              _lib.stream_ptr()))
    return out[:n].cpu().numpy()


def cone_soft_shadow(point, light_direction, octree: DensityOctree, eps: float = 0.01):
    """Blocking in [0,1] from marching the density pyramid toward the light
    (illumination.py:142-155 -> cone_blocking _kernels.py:386-422).  `point` may be
    one point or an (n,3) batch (returns a float or an array accordingly)."""
    torch = _lib.require_device()
    pts = np.asarray(point, dtype=np.float64)
    single = pts.ndim == 1
    pts = np.ascontiguousarray(pts.reshape(-1, 3))
    d = _unit(light_direction, "light direction")
    n = pts.shape[0]
    lod = octree.lod_struct()
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    pts_d = _lib.to_device(pts)
    _lib.check(_lib.lib().lvx_probe_cone(C.byref(lod), _lib.ptr(pts_d), _lib.f64x3(d),
                                         C.c_double(float(eps)), C.c_int64(n), _lib.ptr(out),
                                         _lib.stream_ptr()))
    res = out[:n].cpu().numpy()
    return float(res[0]) if single else res


def ao_density_rays(point, normal, octree: DensityOctree, params: Optional[AOParams] = None):
    """Mean per-ray blocking over deterministic hemisphere rays about the normal,
    each integrating the fine density field until it saturates, leaves the
    radius of influence or exits the grid (illumination.py:176-190)."""
    if params is None:
        params = AOParams()
    torch = _lib.require_device()
    pts = np.asarray(point, dtype=np.float64)
    single = pts.ndim == 1
    pts = np.ascontiguousarray(pts.reshape(-1, 3))
    nrm = np.asarray(normal, dtype=np.float64).reshape(-1, 3)
    nrm = np.stack([_unit(v, "normal") for v in nrm])
    if nrm.shape[0] == 1 and pts.shape[0] > 1:
        nrm = np.repeat(nrm, pts.shape[0], axis=0)
    n = pts.shape[0]
    lod = octree.lod_struct()
    dirs = fibonacci_dirs_device(params.n_rays, 1)
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    pts_d, nrm_d = _lib.to_device(pts), _lib.to_device(np.ascontiguousarray(nrm))
    _lib.check(_lib.lib().lvx_probe_ao_density(
        C.byref(lod), _lib.ptr(pts_d), _lib.ptr(nrm_d), C.c_int32(int(params.n_rays)),
        C.c_double(float(params.radius)), C.c_double(float(params.step)), _lib.ptr(dirs),
        C.c_int64(n), _lib.ptr(out), _lib.stream_ptr()))
    res = out[:n].cpu().numpy()
    return float(res[0]) if single else res


def ao_bake_device(model: VoxelModel, octree: DensityOctree, params: AOParams):
    """The bake kernel on device-resident inputs; returns the f32[V] device tensor."""
    torch = _lib.require_device()
    dirs = fibonacci_dirs_device(params.n_rays, 0)
    out = torch.empty(model.voxel_count, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().lvx_ao_bake(
        _lib.ptr(model.dev("counts")), _lib.i32x3(model.spec.dims), C.c_int32(int(params.n_rays)),
        C.c_double(float(params.radius)), C.c_double(float(params.step)), _lib.ptr(dirs),
        _lib.ptr(octree.flat_device()), _lib.ptr(out), _lib.stream_ptr()))
    return out


def precompute_voxel_ao(model: VoxelModel, octree: DensityOctree, params: Optional[AOParams] = None,
                        workers: int = 1) -> AOField:
    """Full-sphere density-ray occlusion at every occupied voxel centre; defaults
    to 100 rays within 5 voxels at step 1 (illumination.py:193-214).  Unoccupied
    voxels keep 0.  `workers` is accepted for signature compatibility."""
    if params is None:
        params = AOParams(n_rays=100, radius=5.0, step=1.0)
    rx, ry, rz = model.spec.dims
    if tuple(octree.dims(0)) != (rx, ry, rz):
        raise ValueError("octree level 0 does not match the model grid")
    out = ao_bake_device(model, octree, params)
    return AOField(_dev=out, _shape=(rz, ry, rx))


def sample_ao(field: AOField, point, normal=None):
    """Trilinear lookup of the baked field at a grid-space point, clamped to [0,1];
    the normal is accepted for interface parity and ignored (illumination.py:217-225)."""
    pts = np.asarray(point, dtype=np.float64)
    single = pts.ndim == 1
    rz, ry, rx = field.shape
    v = _probe_trilinear(field.flat_device(), 0, (rx, ry, rz), 1.0, pts.reshape(-1, 3))
    v = np.minimum(1.0, np.maximum(0.0, v))
    return float(v[0]) if single else v


def replines_shadow(point, light, replines, grid_dims, level: int = 1, tube_radius: float = 0.3,
                    normal=None) -> int:
    """Like hard_shadow but tested against at most one representative line per coarse voxel
    at the given level; the line's radius is the tube radius scaled to the level and
    thickened by its aggregated weight, clamped to [1,4] (illumination.py:115-139 ->
    replines_ray_blocked, _kernels.py:498-538)."""
    if not 1 <= level < len(replines.levels):
        raise ValueError(f"level must be in [1, {len(replines.levels) - 1}], got {level}")
    torch = _lib.require_device()
    o = _shadow_origin(point, normal)
    to_light = np.asarray(light, dtype=np.float64) - o
    max_t = float(np.linalg.norm(to_light))
    if max_t == 0.0:
        return 1
    d = to_light / max_t
    rep = replines.level_struct(level, grid_dims)
    rays = _lib.to_device(np.concatenate([o, d])[None])
    mt = _lib.to_device(np.asarray([max_t], dtype=np.float64))
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().lvx_probe_replines(C.byref(rep), _lib.ptr(rays), _lib.ptr(mt),
                                             C.c_double(float(tube_radius) * float(1 << level)), C.c_int64(1),
                                             _lib.ptr(out), _lib.stream_ptr()))
    return 0 if int(out.item()) else 1


def _model_struct(model: VoxelModel) -> "_lib.Model":
    counts_d, offsets_d, rec_d, table_d, occ_d = model.device_view(need_occ=True)
    m = _lib.Model()
    m.rx, m.ry, m.rz = model.spec.dims
    m.counts_d, m.offsets_d = counts_d.data_ptr(), offsets_d.data_ptr()
    m.seg_rec_d, m.table_d = rec_d.data_ptr(), table_d.data_ptr()
    m.nsum_d, m.nmask_d, m.ncell_d = occ_d[0].data_ptr(), occ_d[1].data_ptr(), occ_d[2].data_ptr()
    m._keep = (counts_d, offsets_d, rec_d, table_d, occ_d)
    return m


def _shadow_origin(point, normal) -> np.ndarray:
    p = np.asarray(point, dtype=np.float64)
    if normal is None:
        return p
    return p + 1e-3 * _unit(normal, "normal")


def hard_shadow(point, light, model: VoxelModel, radius: float = 0.3, normal=None,
                joint_spheres: bool = True) -> int:
    """1 if the point sees the light position, 0 if any tube or joint sphere lies
    strictly between (illumination.py:96-112 -> geometry_ray_blocked,
    _kernels.py:450-495).  Passing the surface normal offsets the ray origin by 1e-3
    along it."""
    torch = _lib.require_device()
    o = _shadow_origin(point, normal)
    to_light = np.asarray(light, dtype=np.float64) - o
    max_t = float(np.linalg.norm(to_light))
    if max_t == 0.0:
        return 1
    d = to_light / max_t
    m = _model_struct(model)
    rays = _lib.to_device(np.concatenate([o, d])[None])
    mt = _lib.to_device(np.asarray([max_t], dtype=np.float64))
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().lvx_probe_blocked(C.byref(m), _lib.ptr(rays), _lib.ptr(mt), C.c_double(float(radius)),
                                            C.c_int32(1 if joint_spheres else 0), C.c_int64(1), _lib.ptr(out),
                                            _lib.stream_ptr()))
    return 0 if int(out.item()) else 1


def ao_hemisphere_geometry(point, normal, model: VoxelModel, params: Optional[AOParams] = None,
                           tube_radius: float = 0.3, jitter: float = 0.0):
    """Fraction of deterministic hemisphere rays around the normal that hit a tube within
    the radius of influence (illumination.py:158-173 -> ao_hemisphere_point,
    _kernels.py:572-589).  `point` may be one point or an (n,3) array."""
    if params is None:
        params = AOParams()
    torch = _lib.require_device()
    pts = np.asarray(point, dtype=np.float64)
    single = pts.ndim == 1
    pts = np.ascontiguousarray(pts.reshape(-1, 3))
    nrm = np.asarray(normal, dtype=np.float64).reshape(-1, 3)
    nrm = np.stack([_unit(v, "normal") for v in nrm])
    if nrm.shape[0] == 1 and pts.shape[0] > 1:
        nrm = np.repeat(nrm, pts.shape[0], axis=0)
    n = pts.shape[0]
    m = _model_struct(model)
    dirs = _lib.to_device(_lib.fibonacci_dirs(params.n_rays, 1, float(jitter))) if jitter else \
        fibonacci_dirs_device(params.n_rays, 1)
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    pts_d, nrm_d = _lib.to_device(pts), _lib.to_device(np.ascontiguousarray(nrm))
    _lib.check(_lib.lib().lvx_probe_ao_hemisphere(
        C.byref(m), _lib.ptr(pts_d), _lib.ptr(nrm_d), C.c_int32(int(params.n_rays)),
        C.c_double(float(params.radius)), _lib.ptr(dirs), C.c_double(float(tube_radius)), C.c_int64(n),
        _lib.ptr(out), _lib.stream_ptr()))
    v = out[:n].cpu().numpy()
    return float(v[0]) if single else v
