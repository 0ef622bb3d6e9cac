"""Synthetic line sets used by the parity tests and bench.py.

The generators are the ones SURVEY.md section 8(d) defines (and that were run
against the reference while surveying): seeded numpy streams, already in
grid-local units.  Each returns (points (P,3) f64, attrs (P,) f64,
curve_offsets (n+1,) i64) -- the flat batch layout the C-ABI consumes -- and
`as_curveset` lifts that into the reference-style CurveSet.
"""
from __future__ import annotations

import numpy as np


def helices(n: int, pts_per_line: int, dims, seed: int = 1234):
    dx, dy, dz = (float(d) for d in dims)
    rng = np.random.default_rng(seed)
    R = rng.uniform(0.05, 0.45, n) * min(dx, dy)
    ph = rng.uniform(0.0, 2.0 * np.pi, n)
    turns = rng.uniform(0.5, 3.0, n)
    z0 = rng.uniform(0.02, 0.3, n) * dz
    z1 = rng.uniform(0.7, 0.98, n) * dz
    t = np.linspace(0.0, 1.0, pts_per_line)
    ang = ph[:, None] + 2.0 * np.pi * turns[:, None] * t[None, :]
    pts = np.empty((n, pts_per_line, 3))
    pts[..., 0] = dx / 2 + R[:, None] * np.cos(ang)
    pts[..., 1] = dy / 2 + R[:, None] * np.sin(ang)
    pts[..., 2] = z0[:, None] + (z1 - z0)[:, None] * t[None, :]
    attrs = np.broadcast_to(t, (n, pts_per_line)).copy()
    off = np.arange(n + 1, dtype=np.int64) * pts_per_line
    return pts.reshape(-1, 3), attrs.reshape(-1), off


def turbulence(n: int, pts_per_line: int, dims, seed: int = 2024, step: float = 0.66,
               wobble: float = 0.35, margin: float = 0.25):
    d = np.asarray(dims, dtype=np.float64)
    rng = np.random.default_rng(seed)
    p = margin + rng.random((n, 3)) * (d - 2 * margin)
    v = rng.normal(size=(n, 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    pts = np.empty((n, pts_per_line, 3))
    pts[:, 0] = p
    for k in range(1, pts_per_line):
        v = v + wobble * rng.normal(size=(n, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        p = p + step * v
        pts[:, k] = p
    span = d - 2 * margin
    pts = margin + np.abs(((pts - margin) % (2 * span)) - span)
    attrs = np.broadcast_to(np.linspace(0.0, 1.0, pts_per_line), (n, pts_per_line)).copy()
    off = np.arange(n + 1, dtype=np.int64) * pts_per_line
    return pts.reshape(-1, 3), attrs.reshape(-1), off


def wiggles(n: int, pts_per_line: int, dims, seed: int = 7, margin: float = 0.3, sigma: float = 0.9):
    """Random polylines folded into the grid interior (cf. the reference's
    tests/test_voxelizer.py:91-101 `wiggle_curve`), as one batch."""
    rng = np.random.default_rng(seed)
    d = np.asarray(dims, dtype=np.float64)
    p0 = margin + rng.random((n, 1, 3)) * (d - 2 * margin)
    steps = rng.normal(0.0, sigma, size=(n, pts_per_line - 1, 3))
    pts = np.concatenate([p0, p0 + np.cumsum(steps, axis=1)], axis=1)
    span = d - 2 * margin
    pts = margin + np.abs(((pts - margin) % (2 * span)) - span)
    attrs = rng.random((n, pts_per_line))
    off = np.arange(n + 1, dtype=np.int64) * pts_per_line
    return pts.reshape(-1, 3), attrs.reshape(-1), off


def lattice_adversarial(n: int, pts_per_line: int, dims, seed: int = 99):
    """Polylines whose vertices sit on half-integer / integer lattice points:
    exact plane hits, reversals on a plane, edge and corner crossings,
    out-of-grid excursions, repeated vertices, ragged lengths (2..pts_per_line)."""
    rng = np.random.default_rng(seed)
    d = np.asarray(dims, dtype=np.int64)
    pts, attrs, off = [], [], [0]
    for _ in range(n):
        m = int(rng.integers(2, pts_per_line + 1))
        p = rng.integers(-2, 2 * (d + 1) + 1, size=(m, 3)).astype(np.float64) * 0.5
        mix = rng.random(m) < 0.35
        p[mix] += rng.normal(0.0, 0.4, size=(int(mix.sum()), 3))
        pts.append(p)
        attrs.append(rng.random(m))
        off.append(off[-1] + m)
    return np.concatenate(pts), np.concatenate(attrs), np.asarray(off, dtype=np.int64)


def as_curveset(pts, attrs, off):
    from .scene_io import Curve, CurveSet
    curves = [Curve(points=pts[off[i]:off[i + 1]], attrs=attrs[off[i]:off[i + 1]])
              for i in range(len(off) - 1)]
    return CurveSet.from_curves(curves)
