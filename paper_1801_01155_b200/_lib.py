"""ctypes binding of liblinevox_b200.so (the C ABI in include/linevox_b200.h).

There is no CPU fallback: if the shared library is missing, or no sm_100-class
device is visible when a compute entry point is called, this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LVX_LIB: developer override to load an experimental build of the same ABI
LIB_PATH = os.environ.get("LVX_LIB") or os.path.join(_HERE, "liblinevox_b200.so")

MAX_LEVELS = 24


class LvxError(RuntimeError):
    """A C-ABI call returned a nonzero status."""


class Camera(C.Structure):
    _fields_ = [("o", C.c_double * 3), ("r", C.c_double * 3), ("u", C.c_double * 3),
                ("f", C.c_double * 3), ("tan_half", C.c_double), ("aspect", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class Model(C.Structure):
    _fields_ = [("rx", C.c_int32), ("ry", C.c_int32), ("rz", C.c_int32), ("n_bins", C.c_int32),
                ("counts_d", C.c_void_p), ("offsets_d", C.c_void_p), ("seg_rec_d", C.c_void_p),
                ("table_d", C.c_void_p), ("nsum_d", C.c_void_p), ("nmask_d", C.c_void_p),
                ("ncell_d", C.c_void_p), ("packed_d", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("tube_r", C.c_double), ("base_alpha", C.c_double), ("tau", C.c_double),
                ("ka", C.c_double), ("kd", C.c_double), ("ks", C.c_double),
                ("shininess", C.c_double), ("light", C.c_double * 3), ("bg", C.c_double * 4),
                ("opacity_mode", C.c_int32), ("neighbor", C.c_int32), ("joints", C.c_int32),
                ("headlight", C.c_int32), ("shadow_mode", C.c_int32), ("ao_mode", C.c_int32),
                ("ao_n_rays", C.c_int32), ("_pad", C.c_int32), ("ao_radius", C.c_double)]


class RepLines(C.Structure):
    _fields_ = [("valid_d", C.c_void_p), ("a_d", C.c_void_p), ("b_d", C.c_void_p), ("w_d", C.c_void_p),
                ("dims", C.c_int32 * 3), ("_pad", C.c_int32), ("size", C.c_double)]


class Lod(C.Structure):
    _fields_ = [("oct_flat_d", C.c_void_p), ("oct_off", C.c_int64 * (MAX_LEVELS + 1)),
                ("oct_dims", C.c_int64 * (MAX_LEVELS * 3)), ("n_levels", C.c_int32),
                ("_pad", C.c_int32), ("ao_flat_d", C.c_void_p), ("ao_dirs_d", C.c_void_p),
                ("rep", RepLines)]


class Tiling(C.Structure):
    _fields_ = [("tile_w", C.c_int32), ("tile_h", C.c_int32), ("tile_first", C.c_int32),
                ("tile_step", C.c_int32), ("compact", C.c_int32), ("_pad", C.c_int32)]


# every symbol include/linevox_b200.h declares (tests check the library exports all)
SYMBOLS = [
    "lvx_abi_version", "lvx_last_error", "lvx_device_check",
    "lvx_mark_curve_starts", "lvx_scan_scratch_bytes", "lvx_voxel_scan",
    "lvx_voxelize_bound", "lvx_voxelize_clip", "lvx_voxelize_compact", "lvx_raw_regroup", "lvx_scan_u16", "lvx_provenance",
    "lvx_build_seg_records", "lvx_decode_packed", "lvx_density_l0", "lvx_density_l0_u32", "lvx_density_l0_packed", "lvx_octree_layout", "lvx_build_octree",
    "lvx_occupancy_dilate", "lvx_neighbor_sums", "lvx_render_scratch_bytes", "lvx_render", "lvx_render_wf_scratch_bytes", "lvx_render_wf", "lvx_render_wf_last_launches",
    "lvx_render_footprint", "lvx_untile", "lvx_untile_all",
    "lvx_fibonacci_dirs", "lvx_ao_bake", "lvx_probe_dda", "lvx_probe_tube", "lvx_probe_sphere",
    "lvx_probe_trilinear", "lvx_probe_cone", "lvx_probe_ao_density", "lvx_probe_blocked",
    "lvx_probe_ao_hemisphere", "lvx_rep_level", "lvx_probe_replines", "lvx_brute_count", "lvx_brute_render",
    "lvx_probe_clip", "lvx_probe_shade", "lvx_probe_rep_line",
]

_lib = None


def lib():
    """The loaded library.  Raises if it was never built (no silent fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a).  This package has no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        L.lvx_last_error.restype = C.c_char_p
        L.lvx_scan_scratch_bytes.restype = C.c_size_t
        L.lvx_scan_scratch_bytes.argtypes = [C.c_int64]
        L.lvx_render_scratch_bytes.restype = C.c_size_t
        L.lvx_render_wf_scratch_bytes.restype = C.c_size_t
        L.lvx_render_wf_scratch_bytes.argtypes = [C.c_void_p, C.c_void_p, C.c_double]
        for name in SYMBOLS:
            fn = getattr(L, name)
            if name not in ("lvx_last_error", "lvx_scan_scratch_bytes", "lvx_render_scratch_bytes",
                            "lvx_render_wf_scratch_bytes"):
                fn.restype = C.c_int
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().lvx_last_error().decode("utf-8", "replace")
        if rc == 1:
            raise ValueError(msg)
        raise LvxError(f"liblinevox_b200 error {rc}: {msg}")


_device_ok = False


def require_device():
    """torch CUDA device + sm_100 check; called at the top of every compute path."""
    global _device_ok
    import torch
    if not _device_ok:
        if not torch.cuda.is_available():
            raise LvxError("no CUDA device: paper_1801_01155_b200 runs on B200 (sm_100a) only "
                           "and has no CPU fallback")
        torch.cuda.init()
        check(lib().lvx_device_check())
        _device_ok = True
    return torch


def stream_ptr():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return C.c_void_p(0)
    return C.c_void_p(t.data_ptr())


def i32x3(v):
    return (C.c_int32 * 3)(int(v[0]), int(v[1]), int(v[2]))


def f64x3(v):
    return (C.c_double * 3)(float(v[0]), float(v[1]), float(v[2]))


_STAGE = {}            # device index -> (pinned uint8 buffers, events)
_STAGE_CHUNK = 32 << 20  # bytes per staging buffer
_STAGE_MIN = 8 << 20     # arrays below this take the driver's pageable path


def _staged_upload(torch, src, dst):
    """Large pageable array -> device through two cached pinned buffers: the host-side copy into
    the pinned buffer (torch's multi-threaded memcpy) of chunk k+1 overlaps the DMA of chunk k.
    The driver's own pageable path is a single-threaded staging copy (~15 GB/s on this box)."""
    dev = torch.cuda.current_device()
    st = _STAGE.get(dev)
    if st is None:
        st = ([torch.empty(_STAGE_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)],
              [torch.cuda.Event(), torch.cuda.Event()])
        _STAGE[dev] = st
    bufs, evs = st
    s8, d8 = src.reshape(-1).view(torch.uint8), dst.reshape(-1).view(torch.uint8)
    n = s8.numel()
    k = 0
    for lo in range(0, n, _STAGE_CHUNK):
        hi = min(lo + _STAGE_CHUNK, n)
        b = k & 1
        if k >= 2:
            evs[b].synchronize()  # the DMA that last read this buffer is done
        bufs[b][:hi - lo].copy_(s8[lo:hi])
        d8[lo:hi].copy_(bufs[b][:hi - lo], non_blocking=True)
        evs[b].record()
        k += 1
    # the buffers are reused by the next call: its first two chunks wait on these events
    evs[0].synchronize()
    evs[1].synchronize()


def to_device(a: np.ndarray, dtype=None, pad: int = 0):
    """Host numpy -> device tensor on the current stream.  numpy memory is pageable: large arrays
    go through cached pinned staging buffers, small ones through the driver's pageable path.
    pad > 0 (1-D arrays): the device buffer is `pad` zeroed elements longer than the array and a view
    of the array's part is returned -- for arrays the kernels read in aligned words past their end
    (the encoded records: include/linevox_b200.h)."""
    torch = require_device()
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.dtype == np.uint32:  # torch's unsigned support is partial: ship the bit pattern
        a = a.view(np.int32)
    elif a.dtype == np.uint16:
        a = a.view(np.int16)
    elif a.dtype == np.uint64:
        a = a.view(np.int64)
    if not a.flags.writeable:
        import warnings
        with warnings.catch_warnings():  # (the tensor is only read: it is copied to the device right away)
            warnings.simplefilter("ignore", UserWarning)
            t = torch.from_numpy(a)
    else:
        t = torch.from_numpy(a)
    if pad:
        if t.dim() != 1:
            raise ValueError("padding is for 1-D arrays")
        buf = torch.empty(t.numel() + int(pad), dtype=t.dtype, device="cuda")
        buf[t.numel():].zero_()
        out = buf[:t.numel()]
        if a.nbytes < _STAGE_MIN or os.environ.get("LVX_H2D") == "pageable":
            out.copy_(t)
        else:
            _staged_upload(torch, t, out)
        return out
    if a.nbytes < _STAGE_MIN or os.environ.get("LVX_H2D") == "pageable":
        return t.to("cuda", non_blocking=False)
    out = torch.empty(t.shape, dtype=t.dtype, device="cuda")
    _staged_upload(torch, t, out)
    return out


def fibonacci_dirs(n: int, hemisphere: int, jitter: float = 0.0) -> np.ndarray:
    out = np.empty((int(n), 3), dtype=np.float64)
    check(lib().lvx_fibonacci_dirs(C.c_int32(int(n)), C.c_int32(int(hemisphere)),
                                   C.c_double(float(jitter)), out.ctypes.data_as(C.c_void_p)))
    return out
