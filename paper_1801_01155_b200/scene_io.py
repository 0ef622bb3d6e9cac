"""Curve-set types of the reference API (scene_io.py:30-107 of the reference):
same fields, same validation, so callers and tests carry over unchanged.

Beyond the reference, a CurveSet can be built from one flat vertex batch
(`CurveSet.from_flat`), which is the layout the device voxelizer consumes; the
per-curve `Curve` objects are then created lazily.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass
class Curve:
    """One polyline: (n,3) float64 vertex positions and (n,) attributes."""

    points: np.ndarray
    attrs: np.ndarray

    def __post_init__(self):
        self.points = np.ascontiguousarray(self.points, dtype=np.float64)
        self.attrs = np.ascontiguousarray(self.attrs, dtype=np.float64)
        if self.points.ndim != 2 or self.points.shape[1] != 3:
            raise ValueError(f"curve points must be (n,3), got {self.points.shape}")
        if self.points.shape[0] < 2:
            raise ValueError("curve needs at least 2 vertices")
        if self.attrs.shape != (self.points.shape[0],):
            raise ValueError("one attribute per vertex required")
        if np.any(self.attrs < 0.0) or np.any(self.attrs > 1.0):
            raise ValueError("attributes must lie in [0,1]")

    def __len__(self) -> int:
        return self.points.shape[0]


class CurveSet:
    """A set of curves plus the tight axis-aligned bound of all vertices."""

    def __init__(self, curves: Optional[list] = None, bbox: Optional[np.ndarray] = None, *,
                 _flat=None):
        self._curves = curves
        self._flat = _flat  # (points (P,3) f64, attrs (P,) f64, offsets (n+1,) i64)
        self.bbox = bbox

    @classmethod
    def from_curves(cls, curves: list) -> "CurveSet":
        if not curves:
            raise ValueError("no curves")
        lo = np.min([c.points.min(axis=0) for c in curves], axis=0)
        hi = np.max([c.points.max(axis=0) for c in curves], axis=0)
        return cls(curves=list(curves), bbox=np.stack([lo, hi]))

    @classmethod
    def from_flat(cls, points, attrs, offsets) -> "CurveSet":
        """Curves stored back to back: curve i is points[offsets[i]:offsets[i+1]]."""
        points = np.ascontiguousarray(points, dtype=np.float64)
        attrs = np.ascontiguousarray(attrs, dtype=np.float64)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        if points.ndim != 2 or points.shape[1] != 3:
            raise ValueError(f"curve points must be (n,3), got {points.shape}")
        if attrs.shape != (points.shape[0],):
            raise ValueError("one attribute per vertex required")
        if offsets.ndim != 1 or offsets.size < 2:
            raise ValueError("no curves")
        if offsets[0] != 0 or offsets[-1] != points.shape[0] or np.any(np.diff(offsets) < 2):
            raise ValueError("curve needs at least 2 vertices")
        if np.any(attrs < 0.0) or np.any(attrs > 1.0):
            raise ValueError("attributes must lie in [0,1]")
        bbox = np.stack([points.min(axis=0), points.max(axis=0)])
        return cls(curves=None, bbox=bbox, _flat=(points, attrs, offsets))

    @property
    def curves(self) -> list:
        if self._curves is None:
            p, a, off = self._flat
            self._curves = [Curve(points=p[off[i]:off[i + 1]], attrs=a[off[i]:off[i + 1]])
                            for i in range(off.size - 1)]
        return self._curves

    def flat(self):
        """(points, attrs, offsets) of all curves concatenated (voxelizer.py:419-425)."""
        if self._flat is None:
            cs = self._curves
            pts = np.concatenate([c.points for c in cs])
            ats = np.concatenate([c.attrs for c in cs])
            off = np.zeros(len(cs) + 1, dtype=np.int64)
            np.cumsum([len(c) for c in cs], out=off[1:])
            return pts, ats, off
        return self._flat

    @property
    def n_curves(self) -> int:
        if self._curves is not None:
            return len(self._curves)
        return int(self._flat[2].size - 1)

    @property
    def n_vertices(self) -> int:
        if self._flat is not None:
            return int(self._flat[0].shape[0])
        return sum(len(c) for c in self._curves)

    def all_points(self) -> np.ndarray:
        return self.flat()[0]


@dataclass(frozen=True)
class GridSpec:
    """Macro voxel grid: dims (r_x, r_y, r_z) and per-face bin resolution N."""

    dims: tuple
    bins_per_axis: int = 32

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        object.__setattr__(self, "dims", dims)
        if len(dims) != 3 or any(d < 1 for d in dims):
            raise ValueError(f"grid dims must be three positive ints, got {dims}")
        n = self.bins_per_axis
        if n < 2 or n > 256 or (n & (n - 1)) != 0:
            raise ValueError(f"bins_per_axis must be a power of two in [2,256], got {n}")

    @property
    def voxel_count(self) -> int:
        dx, dy, dz = self.dims
        return dx * dy * dz

    @property
    def log2_bins(self) -> int:
        return int(self.bins_per_axis).bit_length() - 1


def grid_spec_for(curves: CurveSet, resolution: int, bins_per_axis: int = 32) -> GridSpec:
    """`resolution` voxels along the longest bbox axis, aspect preserved (scene_io.py:110-121)."""
    if resolution < 1:
        raise ValueError("resolution must be >= 1")
    ext = curves.bbox[1] - curves.bbox[0]
    longest = float(ext.max())
    if longest <= 0.0:
        raise ValueError("degenerate bounding box: zero extent on all axes")
    dims = tuple(max(1, int(round(resolution * float(e) / longest))) for e in ext)
    return GridSpec(dims=dims, bins_per_axis=bins_per_axis)
