"""Host-side record operations of the reference API (voxelizer.py:40-169): the integer packer and
the face-bin snap, against an independent bit-string construction (the reference's own test oracle
idea, tests/test_voxelizer.py:24-36) and its known answers.  No GPU needed."""
import numpy as np
import pytest


def bitstring_pack(seg, n_bins):
    lb = n_bins.bit_length() - 1
    fields = [(seg.face_in, 3), (seg.bin_in, 2 * lb), (seg.face_out, 3), (seg.bin_out, 2 * lb),
              (seg.attr_index, 8), (seg.local_line_id, 5)]
    bits = "".join(format(v, f"0{w}b")[::-1] for v, w in fields)  # LSB first
    width = (len(bits) + 7) // 8
    bits = bits.ljust(8 * width, "0")
    return bytes(int(bits[8 * k:8 * k + 8][::-1], 2) for k in range(width))


@pytest.mark.parametrize("n_bins", [2, 4, 8, 16, 32, 64, 128, 256])
def test_pack_unpack_round_trip(n_bins):
    from paper_1801_01155_b200.voxelizer import QuantizedSegment, pack_segment, record_width, unpack_segment
    rng = np.random.default_rng(n_bins)
    assert record_width(n_bins) == {2: 3, 4: 4, 8: 4, 16: 5, 32: 5, 64: 6, 128: 6, 256: 7}[n_bins]
    for _ in range(300):
        seg = QuantizedSegment(int(rng.integers(6)), int(rng.integers(n_bins * n_bins)), int(rng.integers(6)),
                               int(rng.integers(n_bins * n_bins)), int(rng.integers(256)), int(rng.integers(32)))
        data = pack_segment(seg, n_bins)
        assert data == bitstring_pack(seg, n_bins) and len(data) == record_width(n_bins)
        assert unpack_segment(data, n_bins) == seg


def test_pack_rejects_out_of_range_fields():
    from paper_1801_01155_b200.voxelizer import QuantizedSegment, pack_segment, unpack_segment
    ok = dict(face_in=0, bin_in=0, face_out=0, bin_out=0, attr_index=0, local_line_id=0)
    for bad in (dict(face_in=6), dict(face_out=7), dict(bin_in=16), dict(bin_out=-1), dict(attr_index=256),
                dict(local_line_id=32)):
        with pytest.raises(ValueError):
            pack_segment(QuantizedSegment(**{**ok, **bad}), 4)
    with pytest.raises(ValueError):
        unpack_segment(b"\x00" * 3, 4)
    with pytest.raises(ValueError):
        pack_segment(QuantizedSegment(**ok), 3)


def test_quantize_point_on_face_kats():
    """reference tests/test_voxelizer.py:164-167 and the 3-D form."""
    from paper_1801_01155_b200.voxelizer import quantize_point_on_face
    code, c = quantize_point_on_face((0.3, 0.7), 4, 2)
    assert code == 2 and np.array_equal(c, [0.25, 0.75])
    code, q = quantize_point_on_face((1.0, 2.3, 3.7), 0, 32, (1, 2, 3))
    assert code == 9 + 32 * 22 and np.allclose(q, [1.0, 2 + 9.5 / 32, 3 + 22.5 / 32])
    # the reconstructed point moves by at most half a bin per in-face axis
    assert np.abs(q - np.array([1.0, 2.3, 3.7])).max() <= 0.5 / 32
    with pytest.raises(ValueError, match="off face"):
        quantize_point_on_face((1.2, 2.3, 3.7), 0, 32, (1, 2, 3))
    with pytest.raises(ValueError, match="needs its voxel"):
        quantize_point_on_face((1.0, 2.3, 3.7), 0, 32)
    with pytest.raises(ValueError):
        quantize_point_on_face((0.5, 0.5), 6, 32)


def test_export_table_covers_the_reference_names():
    """Every name the reference exports for the hot-path modules (linevox/__init__.py:20-53) resolves here."""
    import paper_1801_01155_b200 as lv
    names = ["Curve", "CurveSet", "GridSpec", "grid_spec_for",
             "QuantizedSegment", "VoxelModel", "build_voxel_model", "clip_curve_to_voxels", "count_duplicates",
             "pack_segment", "quantize_point_on_face", "record_width", "unpack_segment",
             "DensityOctree", "RepLineField", "build_octree", "build_rep_lines", "compute_density_level0",
             "representative_line",
             "Camera", "Frame", "HitRecord", "RenderParams", "composite", "gather_voxel_hits", "intersect_ray_sphere",
             "intersect_ray_tube", "render_frame", "shade_local", "traverse_voxels",
             "AOField", "AOParams", "ao_density_rays", "ao_hemisphere_geometry", "cone_soft_shadow", "hard_shadow",
             "precompute_voxel_ao", "replines_shadow", "sample_ao",
             "brute_force_render", "image_compare", "memory_report"]
    for n in names:
        assert callable(getattr(lv, n)) or isinstance(getattr(lv, n), type), n
