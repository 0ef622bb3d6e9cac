"""Python-level stand-ins for the few `linevox._kernels` entry points the reference's own tests
call directly (tests/test_raycast.py:9,205, tests/test_illumination.py:6,297).  Each routes to
the device probe of the same operation; none is on the frame path.  Calls from inside numba-jitted
test helpers cannot reach these (numba cannot call back into Python), see tests/test_reference_suite.py.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

# mode codes, _kernels.py:43-55
OPACITY_CONSTANT, OPACITY_TRANSFER, OPACITY_DISTANCE = 0, 1, 2
SHADOW_NONE, SHADOW_HARD, SHADOW_REPLINES, SHADOW_CONE = 0, 1, 2, 3
AO_NONE, AO_HEMISPHERE, AO_DENSITY, AO_PRECOMPUTED = 0, 1, 2, 3
MAX_WINDOW_HITS, MAX_PIXEL_HITS, MAX_SEEN = 1024, 8192, 256  # _kernels.py:36-38


def set_threads(n: int) -> int:
    """Accepted for interface parity (_kernels.py:68-71): the device path has no worker count."""
    return 1


def intersect_tube_raw(ox, oy, oz, dx, dy, dz, ax, ay, az, bx, by, bz, radius):
    """_kernels.py:76-134 with float64 endpoints (the all-float64 specialisation)."""
    from .raycast import probe_tubes
    r = probe_tubes(np.array([[ox, oy, oz, dx, dy, dz]], np.float64), np.array([[ax, ay, az]], np.float64),
                    np.array([[bx, by, bz]], np.float64), float(radius), f32_axis=False)[0]
    return bool(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]), float(r[5])


def intersect_sphere_raw(ox, oy, oz, dx, dy, dz, cx, cy, cz, radius):
    from .raycast import probe_spheres
    r = probe_spheres(np.array([[ox, oy, oz, dx, dy, dz]], np.float64), np.array([[cx, cy, cz]], np.float64),
                      float(radius))[0]
    return bool(r[0]), float(r[1]), float(r[2]), float(r[3]), float(r[4]), float(r[5])


def shade_scalar(nx, ny, nz, lx, ly, lz, vx, vy, vz, ka, kd, ks, shininess):
    from .raycast import probe_shade
    return float(probe_shade(np.array([[nx, ny, nz, lx, ly, lz, vx, vy, vz]], np.float64), ka, kd, ks, shininess)[0])


def ao_density_point(px, py, pz, nx, ny, nz, n_rays, radius, step, hemisphere, oct_flat, oct_off, oct_dims,
                     gx, gy, gz):
    """_kernels.py:592-605 on a flat octree as `raycast._octree_args` returns it."""
    from .lod import build_octree
    torch = _lib.require_device()
    dx, dy, dz = (int(v) for v in np.asarray(oct_dims).reshape(-1, 3)[0])
    level0 = np.asarray(oct_flat, dtype=np.float32)[:int(oct_off[1])].reshape(dz, dy, dx)
    oc = build_octree(level0)  # (kept alive until the probe has run)
    lod = oc.lod_struct()
    dirs = _lib.to_device(_lib.fibonacci_dirs(int(n_rays), int(hemisphere)))
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    pts_d = _lib.to_device(np.array([[px, py, pz]], np.float64))
    nrm_d = _lib.to_device(np.array([[nx, ny, nz]], np.float64))
    _lib.check(_lib.lib().lvx_probe_ao_density(
        C.byref(lod), _lib.ptr(pts_d), _lib.ptr(nrm_d), C.c_int32(int(n_rays)), C.c_double(float(radius)),
        C.c_double(float(step)), _lib.ptr(dirs), C.c_int64(1), _lib.ptr(out), _lib.stream_ptr()))
    return float(out.item())
