"""LoD construction: level-0 density and its 2x2x2 mip chain (lod.py:82-119 of the
reference) on the GPU.

    lvx_density_l0    <- compute_density_level0   lod.py:82-94
    lvx_build_octree  <- _coarsen / build_octree  lod.py:97-119

Fields are indexed [z, y, x]; flattened C order equals the voxel linear index
x + rx*(y + ry*z).  `DensityOctree` keeps the whole pyramid in ONE flat device
buffer (the layout `_octree_args`, raycast.py:369-388, marshals for the render
kernel); `levels` are numpy views downloaded on first access.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .voxelizer import VoxelModel


def octree_layout(dims):
    """(offsets i64[L+1], level dims i64[L,3] as dx,dy,dz, L) of the flat pyramid."""
    off = (C.c_int64 * (_lib.MAX_LEVELS + 1))()
    ld = (C.c_int64 * (_lib.MAX_LEVELS * 3))()
    n = C.c_int32(0)
    _lib.check(_lib.lib().lvx_octree_layout(_lib.i32x3(dims), off, ld, C.byref(n)))
    L = n.value
    return (np.asarray(off[:L + 1], dtype=np.int64),
            np.asarray(ld[:3 * L], dtype=np.int64).reshape(L, 3), L)


class DensityOctree:
    """Dense density fields, level 0 at grid resolution, every level half the
    previous per axis (rounded up) down to 1x1x1 (lod.py:27-58)."""

    def __init__(self, levels=None, *, _flat_dev=None, _dims=None):
        if levels is None and _flat_dev is None:
            raise ValueError("need levels")
        self._levels = None if levels is None else [np.asarray(l, dtype=np.float32) for l in levels]
        self._flat_dev = _flat_dev
        if _dims is None:
            dz, dy, dx = self._levels[0].shape
            _dims = (dx, dy, dz)
        self._dims0 = tuple(int(d) for d in _dims)
        self._off, self._ldims, self._n = octree_layout(self._dims0)
        if self._levels is not None and len(self._levels) != self._n:
            raise ValueError(f"expected {self._n} levels for grid {self._dims0}, got {len(self._levels)}")

    @property
    def levels(self) -> list:
        if self._levels is None:
            flat = self._flat_dev.cpu().numpy()
            self._levels = [flat[self._off[l]:self._off[l + 1]].reshape(
                int(self._ldims[l, 2]), int(self._ldims[l, 1]), int(self._ldims[l, 0]))
                for l in range(self._n)]
        return self._levels

    @property
    def n_levels(self) -> int:
        return self._n

    def dims(self, level: int):
        dx, dy, dz = (int(v) for v in self._ldims[level])
        return dx, dy, dz

    def flat_device(self):
        """The flat f32 pyramid on the GPU (uploaded from `levels` if it was built on the host)."""
        if self._flat_dev is None:
            flat = np.concatenate([np.ascontiguousarray(l, dtype=np.float32).reshape(-1)
                                   for l in self._levels])
            self._flat_dev = _lib.to_device(flat)
        return self._flat_dev

    def lod_struct(self, ao_flat_d=None, ao_dirs_d=None) -> "_lib.Lod":
        s = _lib.Lod()
        s.oct_flat_d = self.flat_device().data_ptr()
        for i, v in enumerate(self._off):
            s.oct_off[i] = int(v)
        for i, v in enumerate(self._ldims.reshape(-1)):
            s.oct_dims[i] = int(v)
        s.n_levels = self._n
        s.ao_flat_d = ao_flat_d.data_ptr() if ao_flat_d is not None else None
        s.ao_dirs_d = ao_dirs_d.data_ptr() if ao_dirs_d is not None else None
        return s

    def sample(self, point, level: int) -> float:
        """Trilinear sample at a grid-space point: cell centres carry the values and
        queries clamp to the field edge (lod.py:42-58).  Evaluated by the device
        probe so it is the same arithmetic the kernels use."""
        from .illumination import _probe_trilinear
        dx, dy, dz = self.dims(level)
        return float(_probe_trilinear(self.flat_device(), int(self._off[level]), (dx, dy, dz),
                                      float(1 << level), np.asarray(point, dtype=np.float64)[None])[0])


def density_level0_device(model: VoxelModel, out=None):
    """Level-0 density as a device tensor f32[V] (no host copy); `out` may be the front of an
    octree buffer, so the mip chain reads it in place."""
    torch = _lib.require_device()
    V = model.voxel_count
    if out is None:
        out = torch.empty(V, dtype=torch.float32, device="cuda")
    if model.voxel_binning_is_external():
        return _density_by_seg_voxel(model, out)
    mode = os.environ.get("LVX_DENSITY", "auto")
    if model.records_match_packed() and (mode == "packed" or (mode == "auto" and not model.has_render_caches())):
        # a model that carries only the encoded arrays (a .vxl file): the sum is taken from them,
        # nothing is expanded (bit-identical; with the render records at hand those are faster,
        # the decode costs more issue slots than the 27 bytes per segment it saves)
        table = _lib.to_device(np.ascontiguousarray(model.transfer_table, dtype=np.float32))
        _lib.check(_lib.lib().lvx_density_l0_packed(
            _lib.ptr(model.dev("counts")), _lib.ptr(model.dev("offsets")), _lib.ptr(model.dev("packed")),
            _lib.i32x3(model.spec.dims), C.c_int32(int(model.spec.bins_per_axis)), _lib.ptr(table), _lib.ptr(out),
            _lib.stream_ptr()))
        return out
    counts_d, offsets_d, rec_d, table_d, _ = model.device_view(need_occ=False)
    _lib.check(_lib.lib().lvx_density_l0(_lib.ptr(counts_d), _lib.ptr(offsets_d), _lib.ptr(rec_d),
                                         _lib.ptr(table_d), C.c_int64(V), _lib.ptr(out),
                                         _lib.stream_ptr()))
    return out


def _density_by_seg_voxel(model: VoxelModel, out):
    """compute_density_level0 bins by `seg_voxel` (lod.py:90-93), not by the headers.  For a model
    whose per-segment arrays were supplied by the caller the two need not agree, so the records are
    put into voxel order with a STABLE sort (bincount adds a voxel's weights in segment order) and
    summed by the same kernel over uncapped counts."""
    torch = _lib.require_device()
    V = model.voxel_count
    dx, dy, _ = model.spec.dims
    vox = model.dev("seg_voxel").to(torch.int64)
    lin = vox[:, 0] + dx * (vox[:, 1] + dy * vox[:, 2])
    order = torch.argsort(lin, stable=True)
    S = int(lin.shape[0])
    rec = torch.empty((max(S, 1), 8), dtype=torch.float32, device="cuda")
    a, b = model.dev("seg_a")[order].contiguous(), model.dev("seg_b")[order].contiguous()
    at, li = model.dev("seg_attr")[order].contiguous(), model.dev("seg_lid")[order].contiguous()
    L, st = _lib.lib(), _lib.stream_ptr()
    _lib.check(L.lvx_build_seg_records(_lib.ptr(a), _lib.ptr(b), _lib.ptr(at), _lib.ptr(li), C.c_int64(S),
                                       _lib.ptr(rec), st))
    counts = torch.bincount(lin, minlength=V)
    offsets = (torch.cumsum(counts, 0) - counts).to(torch.int32)
    table = _lib.to_device(np.ascontiguousarray(model.transfer_table, dtype=np.float32))
    counts32 = counts.to(torch.int32)  # (held until the call is queued: a temporary is freed before the launch)
    _lib.check(L.lvx_density_l0_u32(_lib.ptr(counts32), _lib.ptr(offsets), _lib.ptr(rec),
                                    _lib.ptr(table), C.c_int64(V), _lib.ptr(out), st))
    return out


def compute_density_level0(model: VoxelModel) -> np.ndarray:
    """Per-voxel sum of segment length times transfer-table opacity, (rz, ry, rx) f32."""
    dx, dy, dz = model.spec.dims
    _lib.require_device()
    if model.segment_count == 0:
        return np.zeros((dz, dy, dx), dtype=np.float32)
    return density_level0_device(model).cpu().numpy().reshape(dz, dy, dx)


def _octree_from_level0_device(level0_d, dims) -> DensityOctree:
    torch = _lib.require_device()
    off, _, _ = octree_layout(dims)
    flat = torch.empty(int(off[-1]), dtype=torch.float32, device="cuda")
    flat[:int(off[1])].copy_(level0_d.reshape(-1))
    _lib.check(_lib.lib().lvx_build_octree(_lib.ptr(flat), _lib.i32x3(dims), _lib.stream_ptr()))
    return DensityOctree(_flat_dev=flat, _dims=dims)


def build_octree(level0: np.ndarray) -> DensityOctree:
    """Mip chain of a (rz, ry, rx) field down to 1x1x1 (lod.py:113-119)."""
    level0 = np.asarray(level0)
    if level0.ndim != 3 or level0.size == 0:
        raise ValueError(f"need a non-empty 3D field, got shape {level0.shape}")
    _lib.require_device()
    dz, dy, dx = level0.shape
    l0 = _lib.to_device(np.ascontiguousarray(level0, dtype=np.float32).reshape(-1))
    return _octree_from_level0_device(l0, (dx, dy, dz))


def octree_buffer(dims):
    """Uninitialised flat device buffer of all levels (level 0 first)."""
    torch = _lib.require_device()
    off, _, _ = octree_layout(dims)
    return torch.empty(int(off[-1]), dtype=torch.float32, device="cuda"), int(off[1])


def mips_inplace(flat, dims):
    """Levels 1.. of the pyramid from level 0 at the front of `flat` (lvx_build_octree)."""
    _lib.check(_lib.lib().lvx_build_octree(_lib.ptr(flat), _lib.i32x3(dims), _lib.stream_ptr()))


def build_lod(model: VoxelModel) -> DensityOctree:
    """compute_density_level0 + build_octree without leaving the GPU: the density kernel writes
    level 0 straight into the octree buffer, the mip kernels fill the rest."""
    dims = model.spec.dims
    flat, v0 = octree_buffer(dims)
    density_level0_device(model, out=flat[:v0])
    mips_inplace(flat, dims)
    return DensityOctree(_flat_dev=flat, _dims=dims)


# --- representative lines (lod.py:61-79, 122-284) ---------------------------------------------

def representative_line(starts, ends, origin, size: float, n_bins: int):
    """Average the member segments of one (coarse) voxel into a single line (lod.py:141-169):
    members in the given order, the flip rule, the face-bin snap and the summed length, computed
    by the same device code the level kernel runs per parent voxel.  Returns (a, b, weight) in
    grid units, or None without segments."""
    starts = np.asarray(starts, dtype=np.float64).reshape(-1, 3)
    ends = np.asarray(ends, dtype=np.float64).reshape(-1, 3)
    m = starts.shape[0]
    if m == 0:
        return None
    torch = _lib.require_device()
    s_d, e_d = _lib.to_device(starts), _lib.to_device(ends)
    scratch = torch.empty(m, dtype=torch.float64, device="cuda")
    out = torch.empty(7, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().lvx_probe_rep_line(_lib.ptr(s_d), _lib.ptr(e_d), C.c_int64(m),
                                             _lib.f64x3(np.asarray(origin, dtype=np.float64)), C.c_double(float(size)),
                                             C.c_int32(int(n_bins)), _lib.ptr(scratch), _lib.ptr(out),
                                             _lib.stream_ptr()))
    o = out.cpu().numpy()
    return o[0:3].copy(), o[3:6].copy(), float(o[6])


class RepLevel:
    """One representative line per voxel of a coarsened grid (lod.py:61-65): `valid` (V,) bool,
    `a`, `b` (V,3) float32 grid units, `weight` (V,) float32 summed member length.  Built on
    the device; the numpy views are downloaded on first access."""

    def __init__(self, valid_d, a_d, b_d, w_d, dims):
        self._d = (valid_d, a_d, b_d, w_d)
        self.dims = tuple(int(x) for x in dims)
        self._h = {}

    def _host(self, k, i, conv=None):
        if k not in self._h:
            v = self._d[i].cpu().numpy()
            self._h[k] = conv(v) if conv else v
        return self._h[k]

    @property
    def valid(self):
        return self._host("valid", 0, lambda v: v.astype(bool))

    @property
    def a(self):
        return self._host("a", 1)

    @property
    def b(self):
        return self._host("b", 2)

    @property
    def weight(self):
        return self._host("weight", 3)

    def device(self):
        return self._d


class RepLineField:
    """One optional representative line per voxel at every level >= 1 (lod.py:68-79);
    index 0 is None (the fine level keeps its real segments)."""

    def __init__(self, levels):
        self.levels = levels

    def level_dims(self, level: int, octree_dims) -> tuple:
        d = tuple(octree_dims)
        for _ in range(level):
            d = tuple((x + 1) // 2 for x in d)
        return d

    def level_struct(self, level: int, grid_dims) -> "_lib.RepLines":
        """_rep_args (raycast.py:391-402) as the C struct; the level is clamped like there."""
        level = max(1, min(int(level), len(self.levels) - 1))
        lvl = self.levels[level]
        r = _lib.RepLines()
        v, a, b, w = lvl.device()
        r.valid_d, r.a_d, r.b_d, r.w_d = v.data_ptr(), a.data_ptr(), b.data_ptr(), w.data_ptr()
        for i in range(3):
            r.dims[i] = -(-int(grid_dims[i]) // (1 << level))
        r.size = float(1 << level)
        r._keep = (v, a, b, w)
        return r


def build_rep_lines(model: VoxelModel, octree: DensityOctree, adjacency: bool = True) -> RepLineField:
    """Representative lines for every level >= 1 (lod.py:224-284): level 1 averages the model's
    segments grouped into 2x2x2 voxel blocks, each further level the representatives of the
    level below; the weight is the summed member length.  One kernel per level
    (lvx_rep_level), one thread per parent voxel, same member order as the reference."""
    torch = _lib.require_device()
    L, st = _lib.lib(), _lib.stream_ptr()
    counts_d, offsets_d, rec_d, _, _ = model.device_view(need_occ=False)
    n_bins = int(model.spec.bins_per_axis)
    levels = [None]
    child_dims = tuple(int(x) for x in model.spec.dims)
    prev = None
    for level in range(1, octree.n_levels):
        pd = tuple((x + 1) // 2 for x in child_dims)
        V = pd[0] * pd[1] * pd[2]
        valid = torch.empty(V, dtype=torch.uint8, device="cuda")
        a = torch.empty((V, 3), dtype=torch.float32, device="cuda")
        b = torch.empty((V, 3), dtype=torch.float32, device="cuda")
        w = torch.empty(V, dtype=torch.float32, device="cuda")
        if prev is None:
            args = (_lib.ptr(counts_d), _lib.ptr(offsets_d), _lib.ptr(rec_d), None, None, None, None)
        else:
            pv, pa, pb, pw = prev
            args = (None, None, None, _lib.ptr(pv), _lib.ptr(pa), _lib.ptr(pb), _lib.ptr(pw))
        _lib.check(L.lvx_rep_level(_lib.i32x3(child_dims), *args, C.c_int32(level), C.c_int32(n_bins),
                                   C.c_int32(1 if adjacency else 0), _lib.ptr(valid), _lib.ptr(a), _lib.ptr(b),
                                   _lib.ptr(w), st))
        levels.append(RepLevel(valid, a, b, w, pd))
        prev = (valid, a, b, w)
        child_dims = pd
    return RepLineField(levels)
