"""Pins the CPU oracle against the fixtures the UNMODIFIED reference produced at the sizes
bench.py times (tests/golden/make_golden.py: big_c2_1080p*, big_c3_1080p, accept_tornado256, occ_*).
The stored image rows, counters and sha256 digests are the reference's own; the oracle must
reproduce them bit for bit (same IEEE float64 arithmetic, libm pow in both)."""
import ast
import hashlib

import numpy as np
import pytest

from conftest import golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rows_equal(oracle, g, dims, model, levels, tag=""):
    W, H = (int(x) for x in (g["size"] if "size" in g.files else (640, 360)))
    kw = ast.literal_eval(str(g["params" + tag]))
    nb = kw.pop("neighbor_mode") != "off"
    step = int(g["row_step"])
    img, st = oracle.render(oracle.default_camera(dims, W, H), model, levels, neighbor=nb, rows=(0, H, step), **kw)
    want = g["rows" + tag]
    assert np.array_equal(img[::step], want), f"max diff {np.abs(img[::step] - want).max()}"
    return st


@pytest.mark.parametrize("case", ["helices", "turbulence", "lattice", "cap255", "wiggles"])
def test_occupancy_dilated(oracle, case):
    v, g = golden("vox_" + case), golden("occ_" + case)
    m = oracle.build_voxel_model(v["pts"], v["attrs"], v["off"], tuple(int(x) for x in v["dims"]), int(v["n_bins"]))
    assert np.array_equal(oracle.occupancy_dilated(m).reshape(-1), np.asarray(g["occ"]).reshape(-1))


def test_acceptance_tornado_256(oracle):
    """tests/test_acceptance.py:144-169 of the reference: tornado(1000, 250, 42) @ 256^3, 640x360."""
    g = golden("accept_tornado256")
    dims = tuple(int(d) for d in g["dims"])
    m = oracle.build_voxel_model(g["pts"], g["attrs"], g["off"], dims, 32)
    assert m.segment_count == int(g["segments"])
    assert sha(m.packed) == str(g["packed_sha256"]) and sha(m.counts) == str(g["counts_sha256"])
    for tag in ("_opaque", "_alpha25"):
        rows_equal(oracle, g, dims, m, None, tag)


@pytest.mark.parametrize("fixture", ["big_c2_1080p", "big_c2_1080p_own"])
def test_c2_1080p(oracle, fixture):
    from paper_1801_01155_b200 import synth
    g = golden(fixture)
    dims = (128, 128, 128)
    m = oracle.build_voxel_model(*synth.helices(10000, 100, dims), dims, 32)
    assert m.segment_count == int(g["segments"]) == 5355984
    assert sha(m.packed) == str(g["packed_sha256"]) and sha(m.counts) == str(g["counts_sha256"])
    rows_equal(oracle, g, dims, m, None)


def test_c3_1080p(oracle):
    """The frame bench.py times: model, LoD, AO bake digests and every 16th row of the 1080p frame."""
    from paper_1801_01155_b200 import synth
    g = golden("big_c3_1080p")
    dims = (256, 256, 256)
    m = oracle.build_voxel_model(*synth.turbulence(100000, 100, dims), dims, 32)
    assert m.segment_count == int(g["segments"]) == 9683143
    assert sha(m.packed) == str(g["packed_sha256"]) and sha(m.counts) == str(g["counts_sha256"])
    l0 = oracle.compute_density_level0(m)
    assert sha(l0) == str(g["level0_sha256"])
    levels = oracle.build_octree(l0)
    assert [sha(l) for l in levels] == [str(x) for x in g["levels_sha256"]]
    m.ao = oracle.precompute_voxel_ao(m, levels, 100, 5.0, 1.0)
    assert sha(np.asarray(m.ao)) == str(g["ao_sha256"])
    rows_equal(oracle, g, dims, m, levels)
