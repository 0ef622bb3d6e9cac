"""CPU-only checks: the C-ABI library loads and exports every declared symbol, the
host-side mirror of the reference API validates like the reference, and the
product fails loudly (no fallback) without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


@pytest.fixture(scope="module")
def lv():
    import paper_1801_01155_b200 as lv
    return lv


def test_library_exports_every_declared_symbol():
    from paper_1801_01155_b200 import _lib
    header = open(os.path.join(ROOT, "include", "linevox_b200.h")).read()
    declared = set(re.findall(r"\b(lvx_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.SYMBOLS)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert _lib.lib().lvx_abi_version() == 2


def test_host_only_entry_points(lv):
    from paper_1801_01155_b200 import _lib
    from paper_1801_01155_b200.lod import octree_layout
    off, ld, L = octree_layout((256, 256, 256))
    assert L == 9 and off[-1] == sum((256 >> l) ** 3 for l in range(9))
    off, ld, L = octree_layout((7, 5, 9))  # reference tests/test_lod.py:133-137: ceil(log2(max))+1
    assert L == 5 and ld.tolist() == [[7, 5, 9], [4, 3, 5], [2, 2, 3], [1, 1, 2], [1, 1, 1]]
    g = golden("prim_density")
    assert np.array_equal(_lib.fibonacci_dirs(25, 1), g["fib25_hemi"])
    assert np.array_equal(_lib.fibonacci_dirs(100, 0), g["fib100_sphere"])


def test_no_gpu_means_loud_failure(lv):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1801_01155_b200 import _lib, synth
    cs = lv.CurveSet.from_flat(*synth.helices(3, 10, (8, 8, 8)))
    with pytest.raises(_lib.LvxError, match="no CPU fallback"):
        lv.build_voxel_model(cs, lv.GridSpec((8, 8, 8)))
    with pytest.raises(_lib.LvxError):
        lv.build_octree(np.zeros((2, 2, 2), np.float32))
    assert _lib.lib().lvx_device_check() == 3  # LVX_E_NO_DEVICE
    assert b"no CPU fallback" in _lib.lib().lvx_last_error()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1801_01155_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("brute-force oracle", ""), f


def test_record_width_and_unpack(lv):
    # reference tests/test_voxelizer.py:106-109, tests/test_model_io.py:68
    assert [lv.record_width(n) for n in (2, 4, 8, 16, 32, 64, 128, 256)] == [3, 4, 4, 5, 5, 6, 6, 7]
    for bad in (0, 1, 3, 48, 512):
        with pytest.raises(ValueError):
            lv.record_width(bad)
    # independent bit-string packer (cf. tests/test_voxelizer.py:24-36)
    rng = np.random.default_rng(3)
    for n in (2, 4, 32, 256):
        lb = n.bit_length() - 1
        w = lv.record_width(n)
        recs, fields = [], []
        for _ in range(200):
            f = dict(face_in=int(rng.integers(6)), bin_in=int(rng.integers(n * n)), face_out=int(rng.integers(6)),
                     bin_out=int(rng.integers(n * n)), attr=int(rng.integers(256)), lid=int(rng.integers(32)))
            bits = ""
            for key, width in (("face_in", 3), ("bin_in", 2 * lb), ("face_out", 3), ("bin_out", 2 * lb),
                               ("attr", 8), ("lid", 5)):
                bits += format(f[key], f"0{width}b")[::-1]  # LSB first
            bits = bits.ljust(8 * w, "0")
            recs.append(bytes(int(bits[8 * k:8 * k + 8][::-1], 2) for k in range(w)))
            fields.append(f)
        u = lv.unpack_records(np.frombuffer(b"".join(recs), np.uint8), n)
        for key in ("face_in", "bin_in", "face_out", "bin_out", "attr", "lid"):
            assert u[key].tolist() == [f[key] for f in fields], (n, key)
    # and against the reference's packed bytes
    g = golden("vox_turbulence")
    u = lv.unpack_records(g["packed"], int(g["n_bins"]))
    assert np.array_equal(u["face_in"], g["seg_face_in"]) and np.array_equal(u["bin_out"], g["seg_bin_out"])
    assert np.array_equal(u["attr"], g["seg_attr"]) and np.array_equal(u["lid"], g["seg_lid"])


def test_types_validate_like_the_reference(lv):
    with pytest.raises(ValueError):
        lv.GridSpec((4, 4))
    with pytest.raises(ValueError):
        lv.GridSpec((4, 0, 4))
    with pytest.raises(ValueError):
        lv.GridSpec((4, 4, 4), bins_per_axis=24)
    assert lv.GridSpec((3, 4, 5)).voxel_count == 60 and lv.GridSpec((3, 4, 5), 16).log2_bins == 4
    with pytest.raises(ValueError):
        lv.Curve(points=np.zeros((1, 3)), attrs=np.zeros(1))
    with pytest.raises(ValueError):
        lv.Curve(points=np.zeros((2, 3)), attrs=np.array([0.0, 1.5]))
    with pytest.raises(ValueError):
        lv.CurveSet.from_flat(np.zeros((3, 3)), np.zeros(3), np.array([0, 1, 3]))
    for kw in (dict(tube_radius=0.0), dict(tube_radius=0.6), dict(opacity_mode="x"), dict(base_opacity=0.0),
               dict(tau=1.5), dict(neighbor_mode="maybe"), dict(shadow_mode="x"), dict(ao_mode="x"),
               dict(background=(0, 0, 0))):
        with pytest.raises(ValueError):
            lv.RenderParams(**kw)
    with pytest.raises(ValueError):
        lv.Camera(position=(0, 0, 0), target=(0, 0, 0))
    with pytest.raises(ValueError):
        lv.Camera(position=(0, 0, 0), target=(0, 0, 1), up=(0, 0, 1))
    with pytest.raises(ValueError):
        lv.Camera(position=(0, 0, 0), target=(1, 0, 0), fov=180.0)
    for kw in (dict(n_rays=0), dict(radius=0.0), dict(step=-1.0), dict(mode="x")):
        with pytest.raises(ValueError):
            lv.AOParams(**kw)
    with pytest.raises(ValueError):
        lv.AOField(np.zeros((4, 4), np.float32))


def test_camera_matches_reference_default(lv):
    cam = lv.default_camera((64, 64, 64), 256, 256)
    assert np.allclose(cam.position, [32.0, 32.0 - 1.9 * 64, 32.0 + 0.42 * 1.9 * 64])
    o, d = cam.ray(128, 128)
    assert abs(np.linalg.norm(d) - 1.0) < 1e-12 and np.array_equal(o, cam.position)
    from paper_1801_01155_b200.raycast import camera_struct
    s = camera_struct(cam)
    assert s.tan_half == float(np.tan(np.radians(45.0) * 0.5)) and s.aspect == 1.0


def test_curveset_flat_round_trip(lv):
    from paper_1801_01155_b200 import synth
    pts, attrs, off = synth.wiggles(7, 9, (5, 5, 5))
    a = lv.CurveSet.from_flat(pts, attrs, off)
    b = lv.CurveSet.from_curves(a.curves)
    for x, y in zip(a.flat(), b.flat()):
        assert np.array_equal(x, y)
    assert a.n_curves == 7 and b.n_vertices == 63 and np.array_equal(a.bbox, b.bbox)
    spec = lv.grid_spec_for(a, 16)
    assert max(spec.dims) == 16


def test_model_container_without_gpu(lv):
    g = golden("vox_helices")
    spec = lv.GridSpec(tuple(int(x) for x in g["dims"]), int(g["n_bins"]))
    m = lv.VoxelModel(spec=spec, counts=g["counts"], offsets=g["offsets"], packed=g["packed"],
                      transfer_table=lv.default_transfer_table(), seg_voxel=g["seg_voxel"], seg_a=g["seg_a"],
                      seg_b=g["seg_b"], seg_attr=g["seg_attr"], seg_lid=g["seg_lid"],
                      seg_face_in=g["seg_face_in"], seg_bin_in=g["seg_bin_in"],
                      seg_face_out=g["seg_face_out"], seg_bin_out=g["seg_bin_out"])
    assert m.segment_count == g["seg_attr"].shape[0] and m.record_width == 5
    assert m.memory_bytes == 5 * spec.voxel_count + 5 * m.segment_count
    assert m.linear_index((1, 2, 3)) == 1 + 16 * (2 + 16 * 3)
    assert m.seg_curve is None and m.ao is None
    assert lv.count_duplicates(m) >= 0.0
    m.ao = np.zeros((16, 16, 16), np.float32)
    assert m.ao.shape == (16, 16, 16)
