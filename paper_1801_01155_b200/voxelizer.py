"""Voxelizer front end: the reference's `build_voxel_model` (voxelizer.py:397-488)
with the clip / quantize / sort / pack pipeline running as sm_100a kernels.

The device pipeline (include/linevox_b200.h):

    lvx_mark_curve_starts -> lvx_voxelize_bound -> lvx_voxelize_clip -> lvx_voxel_scan
        -> lvx_raw_regroup -> lvx_voxelize_compact -> lvx_scan_u16 + lvx_provenance

`VoxelModel` keeps the reference's field names.  Arrays live on the GPU; the
numpy views the reference exposes (`model.counts`, `model.packed`, `model.seg_a`,
...) are downloaded on first access and cached.  Assigning a new array to one of
those attributes replaces it and drops the stale device mirror; arrays mutated
*in place* need an explicit `model.invalidate_device()`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _lib
from .scene_io import Curve, CurveSet, GridSpec

_FACE_BITS, _ATTR_BITS, _LID_BITS = 3, 8, 5

# name -> (numpy dtype, trailing shape)
_ARRAY_FIELDS = {
    "counts": (np.uint8, ()), "offsets": (np.uint32, ()), "packed": (np.uint8, ()),
    "seg_voxel": (np.int32, (3,)), "seg_a": (np.float32, (3,)), "seg_b": (np.float32, (3,)),
    "seg_attr": (np.uint8, ()), "seg_lid": (np.uint8, ()),
    "seg_face_in": (np.uint8, ()), "seg_bin_in": (np.uint16, ()),
    "seg_face_out": (np.uint8, ()), "seg_bin_out": (np.uint16, ()),
    "seg_curve": (np.int32, ()), "seg_order": (np.int32, ()),
}
# arrays the render inputs are derived from: the per-segment caches, or -- for a model that
# carries only the encoded arrays (a .vxl file) -- the packed records they are decoded from
_RENDER_INPUTS = ("counts", "offsets", "packed", "seg_a", "seg_b", "seg_attr", "seg_lid")


def _check_bins(n_bins: int) -> int:
    n = int(n_bins)
    if n < 2 or n > 256 or (n & (n - 1)) != 0:
        raise ValueError(f"bin resolution must be a power of two in [2,256], got {n_bins}")
    return n


def record_width(n_bins: int) -> int:
    """Bytes per packed record: ceil((2*(3 + 2*log2 N) + 8 + 5) / 8) (voxelizer.py:70-76)."""
    n = _check_bins(n_bins)
    lb = n.bit_length() - 1
    return (2 * (_FACE_BITS + 2 * lb) + _ATTR_BITS + _LID_BITS + 7) // 8


def unpack_records(packed: np.ndarray, n_bins: int) -> dict:
    """Host-side decode of packed records into their six fields (the layout of
    voxelizer.py:79-89, LSB first).  Used by tests and by callers that want to
    inspect a model without the per-segment caches."""
    n = _check_bins(n_bins)
    w = record_width(n)
    lb = n.bit_length() - 1
    bb = 2 * lb
    raw = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1, w)
    value = np.zeros(raw.shape[0], dtype=np.uint64)
    for k in range(w):
        value |= raw[:, k].astype(np.uint64) << np.uint64(8 * k)
    mask = np.uint64((1 << bb) - 1)

    def field(shift, m):
        return (value >> np.uint64(shift)) & np.uint64(m)

    return {
        "face_in": field(0, 7).astype(np.uint8),
        "bin_in": (field(3, int(mask))).astype(np.uint16),
        "face_out": field(3 + bb, 7).astype(np.uint8),
        "bin_out": field(6 + bb, int(mask)).astype(np.uint16),
        "attr": field(6 + 2 * bb, 0xFF).astype(np.uint8),
        "lid": field(14 + 2 * bb, 0x1F).astype(np.uint8),
    }


# --- the reference's small record / clipping operations (voxelizer.py:40-169, 273-287) -----------
#
# Same names, arguments and error behaviour, so the reference's tests/test_voxelizer.py can be
# pointed at this package.  The integer packer and the bin snap are scalar host operations in
# the reference too; `clip_curve_to_voxels` runs the device clipper (lvx_probe_clip).

@dataclass(frozen=True)
class QuantizedSegment:
    """The six fields of one packed record (voxelizer.py:40-50)."""

    face_in: int
    bin_in: int
    face_out: int
    bin_out: int
    attr_index: int
    local_line_id: int


class ClippedSegment(NamedTuple):
    voxel: tuple
    entry: np.ndarray
    exit: np.ndarray
    attr_entry: float
    attr_exit: float


def _bit_offsets(n: int):
    """LSB-first layout face_in(3) bin_in(2 lb) face_out(3) bin_out(2 lb) attr(8) lid(5)
    (voxelizer.py:79-89): (bin bits, bin_in, face_out, bin_out, attr, lid offsets)."""
    bb = 2 * (n.bit_length() - 1)
    return bb, _FACE_BITS, _FACE_BITS + bb, 2 * _FACE_BITS + bb, 2 * _FACE_BITS + 2 * bb, \
        2 * _FACE_BITS + 2 * bb + _ATTR_BITS


def pack_segment(seg: QuantizedSegment, n_bins: int) -> bytes:
    """One record as `record_width(n_bins)` little-endian bytes (voxelizer.py:92-113)."""
    n = _check_bins(n_bins)
    if not (0 <= seg.face_in < 6 and 0 <= seg.face_out < 6):
        raise ValueError(f"face IDs must be in [0,6), got {seg.face_in}/{seg.face_out}")
    if not (0 <= seg.bin_in < n * n and 0 <= seg.bin_out < n * n):
        raise ValueError(f"bin codes must be in [0,{n * n}), got {seg.bin_in}/{seg.bin_out}")
    if not 0 <= seg.attr_index < 256:
        raise ValueError(f"attr_index out of byte range: {seg.attr_index}")
    if not 0 <= seg.local_line_id < 32:
        raise ValueError(f"local_line_id needs 5 bits: {seg.local_line_id}")
    _, o_bi, o_fo, o_bo, o_at, o_lid = _bit_offsets(n)
    word = (int(seg.face_in) | (int(seg.bin_in) << o_bi) | (int(seg.face_out) << o_fo) | (int(seg.bin_out) << o_bo)
            | (int(seg.attr_index) << o_at) | (int(seg.local_line_id) << o_lid))
    return word.to_bytes(record_width(n), "little")


def unpack_segment(data: bytes, n_bins: int) -> QuantizedSegment:
    """Inverse of pack_segment (voxelizer.py:116-130)."""
    n = _check_bins(n_bins)
    w = record_width(n)
    if len(data) != w:
        raise ValueError(f"expected a {w}-byte record for N={n}, got {len(data)} bytes")
    f = unpack_records(np.frombuffer(bytes(data), dtype=np.uint8), n)
    return QuantizedSegment(face_in=int(f["face_in"][0]), bin_in=int(f["bin_in"][0]), face_out=int(f["face_out"][0]),
                            bin_out=int(f["bin_out"][0]), attr_index=int(f["attr"][0]), local_line_id=int(f["lid"][0]))


_ON_FACE_TOL = 1e-6  # voxelizer.py:36


def quantize_point_on_face(p, face: int, n_bins: int, voxel=None):
    """Snap a face point to the centre of its N x N bin (voxelizer.py:133-169): `p` is either the
    two in-face coordinates or a 3-D grid point with its voxel.  Returns (bin code, snapped point)."""
    n = _check_bins(n_bins)
    if not 0 <= face < 6:
        raise ValueError(f"face ID must be in [0,6), got {face}")
    axis, side = face >> 1, float(face & 1)
    ua, va = (1 if axis == 0 else 0), (1 if axis == 2 else 2)  # in-face axes, ascending
    p = np.asarray(p, dtype=np.float64)
    if p.shape == (2,):
        u, v = p
    elif p.shape == (3,):
        if voxel is None:
            raise ValueError("a 3D point needs its voxel")
        local = p - np.asarray(voxel, dtype=np.float64)
        if abs(local[axis] - side) > _ON_FACE_TOL:
            raise ValueError(f"point {p.tolist()} is {abs(local[axis] - side):.2e} off face {face}")
        if np.any(local < -_ON_FACE_TOL) or np.any(local > 1 + _ON_FACE_TOL):
            raise ValueError(f"point {p.tolist()} lies outside voxel {voxel}")
        u, v = local[ua], local[va]
    else:
        raise ValueError(f"expected a 2D in-face or 3D grid point, got shape {p.shape}")
    bu = min(max(int(np.floor(u * n)), 0), n - 1)
    bv = min(max(int(np.floor(v * n)), 0), n - 1)
    cu, cv = (bu + 0.5) / n, (bv + 0.5) / n
    if p.shape == (2,):
        return bu + n * bv, np.array([cu, cv])
    q = np.empty(3)
    q[axis], q[ua], q[va] = side, cu, cv
    return bu + n * bv, q + np.asarray(voxel, dtype=np.float64)


def clip_batch_device(pts, attrs, off, dims):
    """_clip_batch (voxelizer.py:213-263) on the device: (vox i64[n,3], p_in, p_out f64[n,3], a_in,
    a_out f64[n], key u64[n]) in the reference's chord order."""
    torch = _lib.require_device()
    L, st = _lib.lib(), _lib.stream_ptr()
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    P = pts.shape[0]
    pts_d, attrs_d = _lib.to_device(pts), _lib.to_device(np.ascontiguousarray(attrs, dtype=np.float64))
    off = np.ascontiguousarray(off, dtype=np.int64)
    first = torch.empty(max(P, 1), dtype=torch.uint8, device="cuda")
    off_dev = _lib.to_device(off)  # (held until the call is queued: a temporary is freed before the launch)
    _lib.check(L.lvx_mark_curve_starts(_lib.ptr(off_dev), C.c_int64(off.size - 1), C.c_int64(P),
                                       _lib.ptr(first), st))
    bound = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(L.lvx_voxelize_bound(_lib.ptr(pts_d), _lib.ptr(first), C.c_int64(P), _lib.ptr(bound), st))
    cap = max(int(bound.item()), 1)
    vox = torch.empty((cap, 3), dtype=torch.int64, device="cuda")
    p_in = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    p_out = torch.empty((cap, 3), dtype=torch.float64, device="cuda")
    att = torch.empty((cap, 2), dtype=torch.float64, device="cuda")
    key = torch.empty(cap, dtype=torch.int64, device="cuda")
    n_d = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(L.lvx_probe_clip(_lib.ptr(pts_d), _lib.ptr(attrs_d), _lib.ptr(first), C.c_int64(P),
                                _lib.i32x3(dims), C.c_uint64(cap), _lib.ptr(vox), _lib.ptr(p_in), _lib.ptr(p_out),
                                _lib.ptr(att), _lib.ptr(key), _lib.ptr(n_d), st))
    n = int(n_d.item())
    order = torch.argsort(key[:n])
    g = lambda t: t[:n][order].cpu().numpy()
    a = g(att)
    return g(vox), g(p_in), g(p_out), a[:, 0].copy(), a[:, 1].copy(), g(key).view(np.uint64)


def clip_curve_to_voxels(curve: Curve, spec: GridSpec) -> list:
    """Split one curve into per-voxel chords between face crossings (voxelizer.py:273-287)."""
    n = len(curve)
    vox, p_in, p_out, a_in, a_out, _ = clip_batch_device(curve.points, curve.attrs, np.array([0, n], np.int64), spec.dims)
    return [ClippedSegment(tuple(int(x) for x in vox[i]), p_in[i], p_out[i], float(a_in[i]), float(a_out[i]))
            for i in range(vox.shape[0])]


def default_transfer_table() -> np.ndarray:
    """Blue-grey-red ramp, opacity 1 (voxelizer.py:292-303)."""
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


_DECODED_FIELDS = ("seg_a", "seg_b", "seg_attr", "seg_lid", "seg_voxel", "seg_face_in", "seg_bin_in",
                   "seg_face_out", "seg_bin_out")


def _array_property(name):
    def get(self):
        return self._get_array(name)

    def set_(self, value):
        self._set_array(name, value)

    return property(get, set_)


class VoxelModel:
    """Compact voxel encoding (`counts`, `offsets`, `packed`: 5V + width*S bytes)
    plus the per-segment caches of the reference's VoxelModel (voxelizer.py:306-355).

    Every array argument may be a numpy array (a model that arrives from the
    host, e.g. decoded from a .vxl file) or a torch CUDA tensor (a model built
    on the device)."""

    def __init__(self, spec: GridSpec, counts, offsets, packed, transfer_table, seg_voxel=None,
                 seg_a=None, seg_b=None, seg_attr=None, seg_lid=None, seg_face_in=None,
                 seg_bin_in=None, seg_face_out=None, seg_bin_out=None, dropped_overflow: int = 0,
                 seg_curve=None, seg_order=None, ao=None):
        self.spec = spec
        self.transfer_table = np.asarray(transfer_table, dtype=np.float32)
        self.dropped_overflow = int(dropped_overflow)
        self._host = {}
        self._dev = {}
        self._derived = {}  # seg_rec, occ, table: device-only render inputs
        self._decoded = set()  # per-segment fields produced by _decode_packed (not user-supplied)
        self._from_pipeline = False  # set by model_from_device: every array came out of the voxelizer
        self._ao = None
        for name, value in (("counts", counts), ("offsets", offsets), ("packed", packed),
                            ("seg_voxel", seg_voxel), ("seg_a", seg_a), ("seg_b", seg_b),
                            ("seg_attr", seg_attr), ("seg_lid", seg_lid),
                            ("seg_face_in", seg_face_in), ("seg_bin_in", seg_bin_in),
                            ("seg_face_out", seg_face_out), ("seg_bin_out", seg_bin_out),
                            ("seg_curve", seg_curve), ("seg_order", seg_order)):
            if value is not None:
                self._set_array(name, value)
        self.ao = ao

    # -- array storage ----------------------------------------------------------
    def _set_array(self, name, value):
        if value is None:
            self._host.pop(name, None)
            self._dev.pop(name, None)
        elif isinstance(value, np.ndarray) or not hasattr(value, "data_ptr"):
            dt, tail = _ARRAY_FIELDS[name]
            arr = np.ascontiguousarray(value, dtype=dt)
            if tail:
                arr = arr.reshape((-1,) + tail)
            self._host[name] = arr
            self._dev.pop(name, None)
        else:
            if name == "packed":
                value = _padded_device_bytes(value)
            self._dev[name] = value
            self._host.pop(name, None)
        self._decoded.discard(name)  # now user-supplied
        if name.startswith("seg_") or name in ("counts", "offsets", "packed"):
            self._from_pipeline = False
        if name in _RENDER_INPUTS:
            self._derived.clear()
            self.__dict__.pop("_occ_dilated", None)
        if name in ("counts", "offsets", "packed"):
            # caches decoded from the old encoded arrays are stale (host mirrors included)
            for k in list(self._decoded):
                self._dev.pop(k, None)
                self._host.pop(k, None)
            self._decoded.clear()

    def _get_array(self, name):
        h = self._host.get(name)
        if h is None:
            d = self._dev.get(name)
            if d is None:
                if name in ("seg_curve", "seg_order"):
                    return None  # optional in the reference too
                if name in _DECODED_FIELDS and self._has("packed"):
                    self._decode_packed(caches=True)
                    d = self._dev[name]
                else:
                    raise AttributeError(f"model carries no {name}")
            h = d.cpu().numpy()
            dt = np.dtype(_ARRAY_FIELDS[name][0])
            if h.dtype != dt:  # u16/u32 travel as same-width signed torch tensors
                h = h.view(dt)
            self._host[name] = h
        return h

    def _has(self, name) -> bool:
        return name in self._host or name in self._dev

    def _decode_packed(self, caches: bool):
        """Expand (counts, offsets, packed) on the device (lvx_decode_packed; the reference
        does this on the host when it loads a .vxl file, model_io.py:151-179, 268-297):
        always the render records, with `caches` also the per-segment cache arrays."""
        torch = _lib.require_device()
        S = self.segment_count
        m = max(S, 1)
        rec = torch.empty((m, 8), dtype=torch.float32, device="cuda")
        out = {}
        if caches:
            out = dict(seg_a=torch.empty((m, 3), dtype=torch.float32, device="cuda"),
                       seg_b=torch.empty((m, 3), dtype=torch.float32, device="cuda"),
                       seg_attr=torch.empty(m, dtype=torch.uint8, device="cuda"),
                       seg_lid=torch.empty(m, dtype=torch.uint8, device="cuda"),
                       seg_voxel=torch.empty((m, 3), dtype=torch.int32, device="cuda"),
                       seg_face_in=torch.empty(m, dtype=torch.uint8, device="cuda"),
                       seg_bin_in=torch.empty(m, dtype=torch.int16, device="cuda"),
                       seg_face_out=torch.empty(m, dtype=torch.uint8, device="cuda"),
                       seg_bin_out=torch.empty(m, dtype=torch.int16, device="cuda"))
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        g = out.get
        if S:
            _lib.check(_lib.lib().lvx_decode_packed(
                _lib.ptr(self.dev("packed")), _lib.ptr(self.dev("counts")), _lib.ptr(self.dev("offsets")),
                _lib.i32x3(self.spec.dims), C.c_int32(self.spec.bins_per_axis), _lib.ptr(g("seg_a")),
                _lib.ptr(g("seg_b")), _lib.ptr(g("seg_attr")), _lib.ptr(g("seg_lid")), _lib.ptr(g("seg_voxel")),
                _lib.ptr(g("seg_face_in")), _lib.ptr(g("seg_bin_in")), _lib.ptr(g("seg_face_out")),
                _lib.ptr(g("seg_bin_out")), _lib.ptr(rec), _lib.ptr(err), _lib.stream_ptr()))
            if int(err.item()) != 0:
                raise ValueError("segment record with face ID > 5")  # model_io.py:277-278
        for k, v in out.items():
            if not self._has(k):
                self._dev[k] = v[:S]
                self._decoded.add(k)
        return rec

    counts = _array_property("counts")
    offsets = _array_property("offsets")
    packed = _array_property("packed")
    seg_voxel = _array_property("seg_voxel")
    seg_a = _array_property("seg_a")
    seg_b = _array_property("seg_b")
    seg_attr = _array_property("seg_attr")
    seg_lid = _array_property("seg_lid")
    seg_face_in = _array_property("seg_face_in")
    seg_bin_in = _array_property("seg_bin_in")
    seg_face_out = _array_property("seg_face_out")
    seg_bin_out = _array_property("seg_bin_out")
    seg_curve = _array_property("seg_curve")
    seg_order = _array_property("seg_order")

    @property
    def ao(self):
        """Optional baked occlusion, (rz, ry, rx) float32 (voxelizer.py:334-335).
        Accepts an ndarray or an AOField; a field baked on the GPU is not copied
        to the host until someone reads this attribute."""
        a = self._ao
        if a is not None and not isinstance(a, np.ndarray):
            return a.values
        return a

    @ao.setter
    def ao(self, value):
        self._derived.pop("ao", None)
        if value is None or hasattr(value, "flat_device"):
            self._ao = value
        else:
            self._ao = np.asarray(value, dtype=np.float32)

    def invalidate_device(self):
        """Forget every device mirror of arrays that also exist on the host (call
        after mutating a host array in place)."""
        for name in list(self._dev):
            if name in self._host:
                del self._dev[name]
        self._derived.clear()
        self.__dict__.pop("_occ_dilated", None)

    def dev(self, name):
        """Device tensor of one array field (uploaded from the host copy if needed)."""
        d = self._dev.get(name)
        if d is None:
            # (the kernels read the encoded records in aligned 8-byte words: up to 7 bytes past the end)
            d = _lib.to_device(self._get_array(name), pad=8 if name == "packed" else 0)
            self._dev[name] = d
        return d

    # -- reference properties -----------------------------------------------------
    @property
    def voxel_count(self) -> int:
        return self.spec.voxel_count

    @property
    def segment_count(self) -> int:
        for store in (self._host, self._dev):
            a = store.get("seg_attr")
            if a is not None:
                return int(a.shape[0])
        p = self._host.get("packed")
        if p is None:
            p = self._dev["packed"]
        return int(p.shape[0]) // self.record_width

    @property
    def record_width(self) -> int:
        return record_width(self.spec.bins_per_axis)

    @property
    def memory_bytes(self) -> int:
        return 5 * self.voxel_count + self.record_width * self.segment_count

    def linear_index(self, voxel) -> int:
        dx, dy, _ = self.spec.dims
        return int(voxel[0] + dx * (voxel[1] + dy * voxel[2]))

    # -- device-side render inputs --------------------------------------------------
    def voxel_binning_is_external(self) -> bool:
        """True when `seg_voxel` was handed in by the caller (not produced by the voxelizer or by
        decoding `packed`): such a model's per-voxel grouping is whatever seg_voxel says, which is
        what the reference's compute_density_level0 bins by (lod.py:90-93)."""
        return (not self._from_pipeline) and self._has("seg_voxel") and "seg_voxel" not in self._decoded \
            and self.segment_count > 0

    def records_match_packed(self) -> bool:
        """True when the per-segment arrays are known to be what `packed` decodes to: the model came
        out of the voxelizer, or it carries only the encoded arrays (anything else was decoded from
        them).  False once a caller has supplied per-segment arrays of their own."""
        if not self._has("packed") or self.segment_count == 0:
            return False
        if self._from_pipeline:
            return True
        return all((not self._has(k)) or k in self._decoded
                   for k in ("seg_a", "seg_b", "seg_attr", "seg_lid", "seg_voxel"))

    def has_render_caches(self) -> bool:
        """True when the per-segment arrays the 32-byte render records are built from are there
        (a model built here, or one whose caches were decoded); False for a model that so far
        carries only the encoded arrays (counts, offsets, packed), e.g. read from a .vxl file."""
        return "seg_rec" in self._derived or all(self._has(k) for k in ("seg_a", "seg_b", "seg_attr", "seg_lid"))

    def device_view(self, need_occ: bool = True, need_rec: bool = True):
        """(counts_d, offsets_d, seg_rec_d, table_d, (nsum_d, nmask_d, ncell_d)) -- the lvx_model
        fields.  need_rec=False: the frame is rendered straight from the encoded records
        (`dev("packed")`), seg_rec_d comes back None and nothing is expanded.  The neighbour grids (27-neighbourhood segment counts / occupancy bits
        over the padded grid; nsum > 0 is the reference's dilated occupancy map) are
        only needed in neighbour mode."""
        torch = _lib.require_device()
        L = _lib.lib()
        st = _lib.stream_ptr()
        d = self._derived
        S = self.segment_count
        if need_rec and "seg_rec" not in d and not all(self._has(k) for k in ("seg_a", "seg_b", "seg_attr", "seg_lid")):
            # only the encoded arrays are there (e.g. a .vxl file) and this caller walks render records
            d["seg_rec"] = self._decode_packed(caches=False)
        if need_rec and "seg_rec" not in d:
            rec = torch.empty((max(S, 1), 8), dtype=torch.float32, device="cuda")
            if S:
                _lib.check(L.lvx_build_seg_records(
                    _lib.ptr(self.dev("seg_a")), _lib.ptr(self.dev("seg_b")),
                    _lib.ptr(self.dev("seg_attr")), _lib.ptr(self.dev("seg_lid")),
                    C.c_int64(S), _lib.ptr(rec), st))
            d["seg_rec"] = rec
        if "table" not in d or d.get("table_src") is not self.transfer_table:
            d["table"] = _lib.to_device(np.ascontiguousarray(self.transfer_table, dtype=np.float32))
            d["table_src"] = self.transfer_table
        if need_occ and "occ" not in d:
            rx, ry, rz = self.spec.dims
            cells = (rx + 2) * (ry + 2) * (rz + 2)
            nsum = torch.empty(cells, dtype=torch.int16, device="cuda")
            nmask = torch.empty(cells, dtype=torch.int32, device="cuda")
            ncell = torch.empty(cells, dtype=torch.int64, device="cuda")
            _lib.check(L.lvx_neighbor_sums(_lib.ptr(self.dev("counts")), _lib.i32x3(self.spec.dims),
                                           _lib.ptr(nsum), _lib.ptr(nmask), _lib.ptr(ncell), st))
            d["occ"] = (nsum, nmask, ncell)
        return (self.dev("counts"), self.dev("offsets"), d.get("seg_rec") if need_rec else None, d["table"], d.get("occ"))

    def occupancy_dilated(self) -> np.ndarray:
        """The reference's `_occupancy_dilated` map (raycast.py:351-366): flat u8 over the
        grid padded by one voxel, 1 where the voxel or any 26-neighbour holds segments."""
        torch = _lib.require_device()
        rx, ry, rz = self.spec.dims
        occ = torch.empty((rx + 2) * (ry + 2) * (rz + 2), dtype=torch.uint8, device="cuda")
        _lib.check(_lib.lib().lvx_occupancy_dilate(_lib.ptr(self.dev("counts")), _lib.i32x3(self.spec.dims),
                                                   _lib.ptr(occ), _lib.stream_ptr()))
        return occ.cpu().numpy()

    def ao_device(self):
        """Flat f32[V] device tensor of the baked AO field, or None."""
        a = self._ao
        if a is None:
            return None
        if not isinstance(a, np.ndarray):
            return a.flat_device()
        d = self._derived
        if "ao" not in d:
            d["ao"] = _lib.to_device(np.ascontiguousarray(a.reshape(-1), dtype=np.float32))
        return d["ao"]


# ---------------------------------------------------------------------------------

def _padded_device_bytes(t, spare: int = 8):
    """A device byte tensor whose storage extends at least `spare` bytes past its end (the kernels
    that decode the encoded records read aligned 8-byte words): the tensor itself when its storage
    already does, else a copy into a longer buffer."""
    import torch
    t = t.reshape(-1)
    if not t.is_contiguous():
        t = t.contiguous()
    end = (t.storage_offset() + t.numel()) * t.element_size()
    if t.untyped_storage().nbytes() - end >= spare:
        return t
    buf = torch.empty(t.numel() + spare, dtype=t.dtype, device=t.device)
    buf[t.numel():].zero_()
    buf[:t.numel()].copy_(t)
    return buf[:t.numel()]


def _scratch(n):
    import torch
    nbytes = int(_lib.lib().lvx_scan_scratch_bytes(C.c_int64(max(int(n), 1))))
    return torch.empty(max(nbytes, 16), dtype=torch.uint8, device="cuda")


def stage_clip(pts_d, attrs_d, off_d, n_curves: int, spec: GridSpec, want_edge_kept: bool):
    """Single-pass clipper: mark curve starts, bound the chord count (one host read, it sizes
    the raw arrays), clip + emit.  Returns (vox_cnt u32[V] uncapped, raw_key, raw_q, raw_lin
    [n_slots] -- one slot per plane crossing, raw_lin = 0xFFFFFFFF where no chord was kept --,
    edge_kept u16[P] or None, err)."""
    torch = _lib.require_device()
    L, st = _lib.lib(), _lib.stream_ptr()
    P = int(pts_d.shape[0])
    first = torch.empty(max(P, 1), dtype=torch.uint8, device="cuda")
    _lib.check(L.lvx_mark_curve_starts(_lib.ptr(off_d), C.c_int64(n_curves), C.c_int64(P),
                                       _lib.ptr(first), st))
    bound = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(L.lvx_voxelize_bound(_lib.ptr(pts_d), _lib.ptr(first), C.c_int64(P), _lib.ptr(bound), st))
    cap = int(bound.item())
    if cap >= 2 ** 32:
        raise MemoryError(f"up to {cap} chords exceed the 32-bit offsets of the voxel headers")
    vox_cnt = torch.zeros(spec.voxel_count, dtype=torch.int32, device="cuda")
    raw_key = torch.empty(max(cap, 1), dtype=torch.int64, device="cuda")
    raw_q = torch.empty(max(cap, 1), dtype=torch.int64, device="cuda")
    raw_lin = torch.empty(max(cap, 1), dtype=torch.int32, device="cuda")
    n_slots_d = torch.zeros(1, dtype=torch.int64, device="cuda")
    edge_kept = torch.empty(max(P, 1), dtype=torch.int16, device="cuda") if want_edge_kept else None
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.check(L.lvx_voxelize_clip(
        _lib.ptr(pts_d), _lib.ptr(attrs_d), _lib.ptr(first), C.c_int64(P), _lib.i32x3(spec.dims),
        C.c_int32(spec.bins_per_axis), C.c_uint64(cap), _lib.ptr(vox_cnt), _lib.ptr(raw_key), _lib.ptr(raw_q),
        _lib.ptr(raw_lin), _lib.ptr(n_slots_d), _lib.ptr(edge_kept), _lib.ptr(err), st))
    # every crossing reserves exactly one slot: n_slots == cap
    return vox_cnt, raw_key[:cap], raw_q[:cap], raw_lin[:cap], edge_kept, err


def stage_regroup(raw_key, raw_q, raw_lin, n_raw: int, cursor):
    """Scatter the raw slots (any order, empty ones skipped) into per-voxel groups of 32-byte
    records through the cursors, which end up pointing at the END of every voxel's range."""
    torch = _lib.require_device()
    grouped = torch.empty((max(n_raw, 1), 4), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().lvx_raw_regroup(_lib.ptr(raw_key), _lib.ptr(raw_q), _lib.ptr(raw_lin),
                                          C.c_int64(int(raw_lin.shape[0])), _lib.ptr(cursor), _lib.ptr(grouped),
                                          _lib.stream_ptr()))
    return grouped


def stage_scan(vox_cnt):
    """Prefix sums over the voxel counters.  Returns (cursor, offsets, counts, n_raw, S);
    reading the two totals is the pipeline's one host synchronisation (it sizes the outputs)."""
    torch = _lib.require_device()
    V = int(vox_cnt.shape[0])
    cursor = torch.empty(V, dtype=torch.int32, device="cuda")
    offsets = torch.empty(V, dtype=torch.int32, device="cuda")  # u32 bit pattern
    counts = torch.empty(V, dtype=torch.uint8, device="cuda")
    totals = torch.zeros(2, dtype=torch.int64, device="cuda")
    scratch = _scratch(V)  # (held until the call is queued: a temporary is freed before the launch)
    _lib.check(_lib.lib().lvx_voxel_scan(_lib.ptr(vox_cnt), C.c_int64(V), _lib.ptr(cursor),
                                         _lib.ptr(offsets), _lib.ptr(counts), _lib.ptr(totals),
                                         _lib.ptr(scratch), _lib.stream_ptr()))
    n_raw, S = (int(x) for x in totals.cpu().tolist())
    if n_raw >= 2 ** 32:
        raise MemoryError(f"{n_raw} chords exceed the 32-bit offsets of the voxel headers")
    return cursor, offsets, counts, n_raw, S


def stage_compact(grouped, n_raw: int, vox_cnt, cursor_end, offsets, counts,
                  spec: GridSpec, S: int, caches: bool, want_keys: bool):
    """Pass 3: per-voxel ordering by key, 255 cap, lid, decode, pack."""
    torch = _lib.require_device()
    w = record_width(spec.bins_per_axis)
    m = max(S, 1)
    dev = "cuda"
    out = {
        "counts": counts, "offsets": offsets,
        # (+ 8: the kernels that decode the records read aligned 8-byte words, up to 7 bytes past the end)
        "packed": torch.empty(m * w + 8, dtype=torch.uint8, device=dev)[:m * w],
        "seg_rec": torch.empty((m, 8), dtype=torch.float32, device=dev),
    }
    if caches:
        out.update(
            seg_a=torch.empty((m, 3), dtype=torch.float32, device=dev),
            seg_b=torch.empty((m, 3), dtype=torch.float32, device=dev),
            seg_attr=torch.empty(m, dtype=torch.uint8, device=dev),
            seg_lid=torch.empty(m, dtype=torch.uint8, device=dev),
            seg_voxel=torch.empty((m, 3), dtype=torch.int32, device=dev),
            seg_face_in=torch.empty(m, dtype=torch.uint8, device=dev),
            seg_bin_in=torch.empty(m, dtype=torch.int16, device=dev),
            seg_face_out=torch.empty(m, dtype=torch.uint8, device=dev),
            seg_bin_out=torch.empty(m, dtype=torch.int16, device=dev))
    if want_keys:
        out["seg_key"] = torch.empty(m, dtype=torch.int64, device=dev)
    g = out.get
    _lib.check(_lib.lib().lvx_voxelize_compact(
        _lib.ptr(grouped), C.c_int64(n_raw), _lib.ptr(vox_cnt),
        _lib.ptr(cursor_end), _lib.ptr(offsets), _lib.i32x3(spec.dims), C.c_int32(spec.bins_per_axis),
        _lib.ptr(out["packed"]), _lib.ptr(g("seg_a")), _lib.ptr(g("seg_b")), _lib.ptr(g("seg_attr")),
        _lib.ptr(g("seg_lid")), _lib.ptr(g("seg_voxel")), _lib.ptr(g("seg_face_in")),
        _lib.ptr(g("seg_bin_in")), _lib.ptr(g("seg_face_out")), _lib.ptr(g("seg_bin_out")),
        _lib.ptr(g("seg_key")), _lib.ptr(out["seg_rec"]), _lib.stream_ptr()))
    for k in list(out):  # trim the >=1 padding of empty models
        if k not in ("counts", "offsets"):
            out[k] = out[k][:S * w] if k == "packed" else out[k][:S]
    return out


def stage_provenance(seg_key, S: int, edge_kept, off_d, n_curves: int):
    """seg_curve / seg_order (voxelizer.py:254-262, 486-487) from the provenance keys."""
    torch = _lib.require_device()
    seg_curve = torch.empty(S, dtype=torch.int32, device="cuda")
    seg_order = torch.empty(S, dtype=torch.int32, device="cuda")
    if S:
        P = int(edge_kept.shape[0])
        edge_base = torch.empty(P, dtype=torch.int32, device="cuda")
        L, st = _lib.lib(), _lib.stream_ptr()
        scratch = _scratch(P)
        _lib.check(L.lvx_scan_u16(_lib.ptr(edge_kept), C.c_int64(P), _lib.ptr(edge_base),
                                  _lib.ptr(scratch), st))
        _lib.check(L.lvx_provenance(_lib.ptr(seg_key), C.c_int64(S), _lib.ptr(edge_base),
                                    _lib.ptr(off_d), C.c_int64(n_curves), _lib.ptr(seg_curve),
                                    _lib.ptr(seg_order), st))
    return seg_curve, seg_order


def check_budget(spec: GridSpec, S: int, memory_budget: Optional[int]):
    w = record_width(spec.bins_per_axis)
    V = spec.voxel_count
    total_bytes = 5 * V + w * S
    if memory_budget is not None and total_bytes > memory_budget:
        raise MemoryError(f"model needs {total_bytes} bytes (5*{V} + {w}*{S}), "
                          f"budget is {memory_budget}")


def voxelize_device(pts_d, attrs_d, off_d, n_curves: int, spec: GridSpec, *, caches: bool = True,
                    provenance: bool = True, memory_budget: Optional[int] = None):
    """Run the device pipeline on vertex arrays that already live on the GPU.

    pts_d f64[P,3], attrs_d f64[P], off_d i64[n_curves+1].  Returns a dict of
    device tensors plus `dropped` and `n_segments`.  This is the kernel-only path
    bench.py times; `build_voxel_model` wraps it with the host<->device copies."""
    vox_cnt, raw_key, raw_q, raw_lin, edge_kept, err = stage_clip(pts_d, attrs_d, off_d, n_curves, spec,
                                                                  provenance)
    cursor, offsets, counts, n_raw, S = stage_scan(vox_cnt)
    check_budget(spec, S, memory_budget)
    grouped = stage_regroup(raw_key, raw_q, raw_lin, n_raw, cursor)
    del raw_key, raw_q, raw_lin
    out = stage_compact(grouped, n_raw, vox_cnt, cursor, offsets, counts, spec, S, caches, provenance)
    if provenance:
        out["seg_curve"], out["seg_order"] = stage_provenance(out.pop("seg_key"), S, edge_kept,
                                                              off_d, n_curves)
    out["n_segments"] = S
    out["dropped"] = n_raw - S
    out["err"] = err
    return out


def model_from_device(out: dict, spec: GridSpec, transfer_table) -> "VoxelModel":
    if int(out["err"].item()) != 0:
        # voxelizer.py:366-368
        raise AssertionError("chord endpoint off every face")
    g = out.get
    model = VoxelModel(
        spec=spec, counts=out["counts"], offsets=out["offsets"], packed=out["packed"],
        transfer_table=transfer_table, seg_voxel=g("seg_voxel"), seg_a=g("seg_a"),
        seg_b=g("seg_b"), seg_attr=g("seg_attr"), seg_lid=g("seg_lid"),
        seg_face_in=g("seg_face_in"), seg_bin_in=g("seg_bin_in"),
        seg_face_out=g("seg_face_out"), seg_bin_out=g("seg_bin_out"),
        dropped_overflow=out["dropped"], seg_curve=g("seg_curve"), seg_order=g("seg_order"))
    model._derived["seg_rec"] = out["seg_rec"]
    model._from_pipeline = True
    return model


def _check_table(transfer_table):
    if transfer_table is None:
        transfer_table = default_transfer_table()
    transfer_table = np.asarray(transfer_table, dtype=np.float32)
    if transfer_table.shape != (256, 4):
        raise ValueError(f"transfer table must be (256,4), got {transfer_table.shape}")
    return transfer_table


def build_voxel_model(curves: CurveSet, spec: GridSpec, transfer_table=None, workers: int = 1,
                      memory_budget: Optional[int] = None) -> VoxelModel:
    """Clip, quantize, pack and compact a whole curve set (voxelizer.py:397-488).

    `workers` is accepted for signature compatibility: the reference's output
    does not depend on it (voxelizer.py:401-403) and the device pipeline has no
    use for it.  Voxels crossed by more than 255 chords keep the first 255 in
    curve order; the rest are counted in `dropped_overflow`."""
    transfer_table = _check_table(transfer_table)
    _lib.require_device()
    pts, attrs, off = curves.flat()
    pts_d = _lib.to_device(pts, np.float64)
    attrs_d = _lib.to_device(attrs, np.float64)
    off_d = _lib.to_device(off, np.int64)
    out = voxelize_device(pts_d, attrs_d, off_d, int(off.size - 1), spec,
                          memory_budget=memory_budget)
    return model_from_device(out, spec, transfer_table)


def count_duplicates(model: VoxelModel) -> float:
    """Fraction of segments whose (voxel, faces, bins) repeat an earlier record
    (voxelizer.py:491-509)."""
    s = model.segment_count
    if s == 0:
        return 0.0
    dx, dy, _ = model.spec.dims
    v = model.seg_voxel.astype(np.int64)
    lin = v[:, 0] + dx * (v[:, 1] + dy * v[:, 2])
    rows = np.stack([lin, model.seg_face_in.astype(np.int64), model.seg_bin_in.astype(np.int64),
                     model.seg_face_out.astype(np.int64), model.seg_bin_out.astype(np.int64)], axis=1)
    return float(s - np.unique(rows, axis=0).shape[0]) / float(s)
